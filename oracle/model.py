"""oracle/model.py -- TEST INFRASTRUCTURE ONLY.

Pure-Python restatement of the reference's send-method model and profile
format, used as the checker for the product's C++ model (libstridepack_b200:
sp_profile_*, sp_interp_*, sp_model_times, sp_choose_method). float64 with
the same operation order as the reference, so results compare exactly.

Follows /root/reference/proj/include/stridepack/:
  perf_model.hpp:75-97   locate          perf_model.hpp:100-108 mix
  perf_model.hpp:113-122 interp_1d       perf_model.hpp:125-136 interp_2d
  perf_model.hpp:139-159 t_device / t_oneshot / t_staged
  perf_model.hpp:163-179 choose_method   profile_io.hpp:88-164 load_profile
  profile_io.hpp:174-213 save_profile
Pinned by tests/test_model.py against tests/golden/model_golden.json, which
the reference itself produced (tests/golden/make_golden_model.py).
"""
from __future__ import annotations

import math

CURVES = ["cpu_cpu", "gpu_gpu", "d2h", "h2d"]
SURFACES = ["gpu_pack", "gpu_unpack", "host_pack", "host_unpack"]
ONESHOT, DEVICE, STAGED = 0, 1, 2


class EmptyProfile(Exception):
    pass


class ParseError(Exception):
    pass


class InvalidArgument(Exception):
    pass


def locate(xs, q):
    if q <= xs[0]:
        return 0, 0, 0.0
    if q >= xs[-1]:
        return len(xs) - 1, len(xs) - 1, 0.0
    hi = 1
    while xs[hi] < q:
        hi += 1
    if q == xs[hi]:
        return hi, hi, 0.0
    lo = hi - 1
    if q == xs[lo]:
        return lo, lo, 0.0
    return lo, hi, (math.log(q) - math.log(xs[lo])) / (math.log(xs[hi]) - math.log(xs[lo]))


def mix(a, b, u):
    if a == b:
        return a
    if a <= 0.0 or b <= 0.0:
        return (1.0 - u) * a + u * b
    return math.exp((1.0 - u) * math.log(a) + u * math.log(b))


def interp_1d(curve, x):
    sizes, times = curve
    if not sizes:
        raise EmptyProfile("interp_1d: curve has no samples")
    lo, hi, u = locate(sizes, x)
    return times[lo] if lo == hi else mix(times[lo], times[hi], u)


def interp_2d(surf, obj, blk):
    objs, blks, t = surf
    if not objs or not blks:
        raise EmptyProfile("interp_2d: surface has no samples")
    olo, ohi, ou = locate(objs, obj)
    blo, bhi, bu = locate(blks, blk)
    t0 = mix(t[olo][blo], t[ohi][blo], ou)
    t1 = mix(t[olo][bhi], t[ohi][bhi], ou)
    return mix(t0, t1, bu)


def times(p, o, b):
    o, b = float(o), float(b)
    dev = interp_2d(p["gpu_pack"], o, b) + interp_1d(p["gpu_gpu"], o) + interp_2d(p["gpu_unpack"], o, b)
    one = interp_2d(p["host_pack"], o, b) + interp_1d(p["cpu_cpu"], o) + interp_2d(p["host_unpack"], o, b)
    stg = (interp_2d(p["gpu_pack"], o, b) + interp_1d(p["d2h"], o) + interp_1d(p["cpu_cpu"], o)
           + interp_1d(p["h2d"], o) + interp_2d(p["gpu_unpack"], o, b))
    return dev, one, stg


def choose(p, o, b):
    if o <= 0 or b <= 0 or b > o:
        raise InvalidArgument("choose_method: need 0 < block_size <= object_size")
    dev, one, stg = times(p, o, b)
    best, bt = DEVICE, dev
    if one < bt:
        best, bt = ONESHOT, one
    if stg < bt:
        best = STAGED
    return best


def parse(text):
    curves = {n: ([], []) for n in CURVES}
    rows = {}
    cur_c = cur_s = None
    for lineno, line in enumerate(text.split("\n"), 1):
        line = line.split("#", 1)[0]
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "curve":
            if len(tok) < 2 or tok[1] not in curves:
                raise ParseError(f"profile line {lineno}: unknown curve name")
            cur_c, cur_s = tok[1], None
        elif tok[0] == "surface":
            if len(tok) < 2 or tok[1] not in SURFACES:
                raise ParseError(f"profile line {lineno}: unknown surface name")
            cur_s, cur_c = tok[1], None
            rows.setdefault(cur_s, [])
        else:
            try:
                a = float(tok[0])
            except ValueError:
                raise ParseError(f"profile line {lineno}: expected a number")
            if cur_c is not None:
                if len(tok) < 2:
                    raise ParseError(f"profile line {lineno}: curve rows are `size time`")
                curves[cur_c][0].append(a)
                curves[cur_c][1].append(float(tok[1]))
            elif cur_s is not None:
                if len(tok) < 3:
                    raise ParseError(f"profile line {lineno}: surface rows are `object block time`")
                rows[cur_s].append((a, float(tok[1]), float(tok[2])))
            else:
                raise ParseError(f"profile line {lineno}: data row before any section header")
    for n, (s, t) in curves.items():
        for i in range(len(s)):
            if s[i] <= 0 or t[i] < 0 or (i and s[i] <= s[i - 1]):
                raise ParseError(f"profile: curve {n} invalid")
    p = dict(curves)
    for n in SURFACES:
        p[n] = ([], [], [])
    for n, rs in rows.items():
        objs = sorted({r[0] for r in rs})
        blks = sorted({r[1] for r in rs})
        if any(r[0] <= 0 or r[1] <= 0 or r[2] < 0 for r in rs) or len(rs) != len(objs) * len(blks):
            raise ParseError(f"profile: surface {n} invalid")
        grid = [[None] * len(blks) for _ in objs]
        for o, b, t in rs:
            i, j = objs.index(o), blks.index(b)
            if grid[i][j] is not None:
                raise ParseError(f"profile: surface {n} has duplicate points")
            grid[i][j] = t
        p[n] = (objs, blks, grid)
    return p


def save(p, header=""):
    out = []
    if header:
        out += ["# " + h for h in header.split("\n")]
    for n in CURVES:
        out.append(f"curve {n}")
        out += [f"{s:.9e} {t:.9e}" for s, t in zip(*p[n])]
    for n in SURFACES:
        out.append(f"surface {n}")
        objs, blks, t = p[n]
        out += [f"{o:.9e} {b:.9e} {t[i][j]:.9e}" for i, o in enumerate(objs) for j, b in enumerate(blks)]
    return "\n".join(out) + "\n"


def scaled(p, k):
    q = {}
    for n in CURVES:
        q[n] = (list(p[n][0]), [t * k for t in p[n][1]])
    for n in SURFACES:
        objs, blks, t = p[n]
        q[n] = (list(objs), list(blks), [[v * k for v in row] for row in t])
    return q

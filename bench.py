#!/usr/bin/env python3
"""bench.py -- MPI_Pack/MPI_Unpack throughput of the B200 datatype engine.

Workload (BASELINE.json configs[1], "cfg2"): a 3D MPI_Type_create_subarray
of a 1 MiB object in a 1024^3-byte allocation, contiguous-dim extent E0 swept
over 1..512 B (E1, E2 per SURVEY.md §8a). One STEP = for every E0: pack K
objects (incount = K, objects one extent = 1 GiB apart) and unpack them back,
through the product's C-ABI on device-resident buffers. The L2 is flushed
(a 512 MiB write) before every kernel and only the kernels are timed, with
CUDA events on the launching stream.

  value      = algorithmic bytes (2 x incount x size per pack or unpack:
               described bytes read + packed bytes written) / kernel time
  e2e        = the same metric through the same C-ABI with the packed
               message in pinned HOST memory: unpack reads it over PCIe,
               pack writes it back (the paper's one-shot method); host<->
               device traffic is inside the timed region
  roofline   = dominant kernel vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline = the reference's own pack/unpack (oracle/_ref, compiled from
               the untouched reference headers) on this host, bounded sample

--impl reference times the reference CPU executor on the same workload
(bounded: one object per E0 per step) with all host threads.
Multi-GPU: pack/unpack does not shard ("replicas only"): each rank
runs the same workload on its own GPU; value sums over ranks, time is the
max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E0S = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
METRIC = "MPI_Pack/Unpack GB/s (3D subarray, 1 MiB object, E0 sweep 1-512 B)"
UNIT = "GB/s"
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent


def cfg2_dims(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return e0, e1, e2


def cfg2_prog(e0):
    e0, e1, e2 = cfg2_dims(e0)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", FALLBACK_HBM)), "measured"
    return FALLBACK_HBM, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md's clocks line). The timed region is tens of ms, shorter
    than nvidia-smi's sampling period, so the same NVML counters nvidia-smi
    reads are polled from a thread every 2 ms; nvidia-smi -lms is the
    fallback when NVML is unavailable."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.nvml = []  # (sm_mhz, max_mhz, reason_bits)
        self.source = None
        self._stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            uuid = "GPU-" + str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, pynvml, h):
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while True:
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.nvml.append((sm, mx, bits))
            except Exception:
                pass
            if self._stop.wait(0.002):
                break

    def __enter__(self):
        try:
            pynvml, h = self._nvml_handle()
            self.source = "nvml-2ms"
            # the timed loop is a tight Python loop: a short GIL switch
            # interval lets the poller run every ~2 ms inside it, and the
            # region starts only once the poller has taken its first sample
            self._switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0002)
            self.t = threading.Thread(target=self._poll, args=(pynvml, h), daemon=True)
            self.t.start()
            t0 = time.perf_counter()
            while not self.nvml and time.perf_counter() - t0 < 1.0:
                time.sleep(0.001)
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi-100ms"
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self._stop.set()
        if getattr(self, "_switch", None):
            sys.setswitchinterval(self._switch)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self.source:
            self.t.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s_, m_, bits in self.nvml:
            sm.append(float(s_))
            mx = float(m_)
            for n, bit in self.REASONS.items():
                if bits & bit:
                    reasons.add(n)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------ distributed
def dist_setup(n):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, local, world


def reduce_device():
    import torch.distributed as dist
    return "cpu" if dist.is_initialized() and dist.get_backend() == "gloo" else "cuda"


def barrier_max(torch, world, value):
    if world == 1:
        return value
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier_sum(torch, world, value):
    if world == 1:
        return value
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=reduce_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def shared_job_name(world, rank):
    """one name for the engine's node-local runtime, agreed by all ranks"""
    import uuid
    name = ["bench" + uuid.uuid4().hex[:10]]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(name, src=0)
    return name[0]


# ------------------------------------------------------------------ reference CPU
def reference_engine():
    from oracle.pyoracle import reference, oracle
    r = reference()
    if r is not None:
        return r, "reference"
    return oracle(), "port"


def cpu_sample(threads, budget_s, reps_min=1):
    """Times the reference CPU pack+unpack of one cfg2 object per E0 (commit
    excluded). Returns (GB/s, seconds, reps, kind)."""
    import numpy as np
    eng, kind = reference_engine()
    buf = np.zeros(1 << 30, np.uint8)  # the 1024^3 allocation
    buf[::4093] = 7
    total_bytes, total_t, reps = 0, 0.0, 0
    handles = [(e0, eng.handle(cfg2_prog(e0))) for e0 in E0S]
    packed = np.zeros(1 << 20, np.uint8)
    t_start = time.perf_counter()
    while reps < reps_min or (time.perf_counter() - t_start) < budget_s:
        for e0, h in handles:
            t0 = time.perf_counter()
            if kind == "reference":
                st, _ = eng.pack_h(h, buf.ctypes.data, buf.nbytes, 1, packed.ctypes.data, packed.nbytes, 0, threads)
                st2, _ = eng.unpack_h(h, packed.ctypes.data, packed.nbytes, 0, 1, buf.ctypes.data, buf.nbytes, threads)
            else:
                st, _ = eng.pack_h(h, buf.ctypes.data, buf.nbytes, 1, packed.ctypes.data, packed.nbytes, 0)
                st2, _ = eng.unpack_h(h, packed.ctypes.data, packed.nbytes, 0, 1, buf.ctypes.data, buf.nbytes)
            total_t += time.perf_counter() - t0
            assert st == 0 and st2 == 0
            total_bytes += 4 * (1 << 20)
        reps += 1
    return total_bytes / total_t / 1e9, total_t, reps, kind


def reference_sample(eng, kind, handles, K, buf, packed, threads):
    """one step of the reference arm: pack + unpack of K cfg2 objects (one
    extent = 1 GiB apart, as the GPU arm) per E0 through the reference's
    own stridepack::pack/unpack. Returns (algorithmic bytes, seconds)."""
    t, nbytes = 0.0, 0
    for e0, h in handles:
        t0 = time.perf_counter()
        if kind == "reference":
            st, _ = eng.pack_h(h, buf.ctypes.data, buf.nbytes, K, packed.ctypes.data, packed.nbytes, 0, threads)
            st2, _ = eng.unpack_h(h, packed.ctypes.data, packed.nbytes, 0, K, buf.ctypes.data, buf.nbytes, threads)
        else:
            st, _ = eng.pack_h(h, buf.ctypes.data, buf.nbytes, K, packed.ctypes.data, packed.nbytes, 0)
            st2, _ = eng.unpack_h(h, packed.ctypes.data, packed.nbytes, 0, K, buf.ctypes.data, buf.nbytes)
        t += time.perf_counter() - t0
        assert st == 0 and st2 == 0
        nbytes += 2 * 2 * K * (1 << 20)
    return nbytes, t


def run_reference(args):
    """The reference arm on the GPU arm's exact config: cfg2, every E0,
    incount = K objects per call, pack + unpack, all host threads."""
    import numpy as np
    rank, local, world = dist_setup(args.gpus)
    if rank != 0:
        return 0
    threads = 0  # PackOptions{.threads = 0}: hardware concurrency
    ncores = os.cpu_count() or 1
    K = args.incount
    eng, kind = reference_engine()
    buf = np.zeros(K << 30, np.uint8)  # K objects one extent (the 1024^3 allocation) apart, as on the GPU
    packed = np.zeros(K << 20, np.uint8)
    handles = [(e0, eng.handle(cfg2_prog(e0))) for e0 in E0S]
    for _ in range(args.warmup):
        reference_sample(eng, kind, handles, K, buf, packed, threads)
    t_total, b_total = 0.0, 0
    for _ in range(args.steps):
        nb, t = reference_sample(eng, kind, handles, K, buf, packed, threads)
        t_total += t
        b_total += nb
    value = b_total / t_total / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"cfg2: MPI_Type_create_subarray 3D, 1 MiB object in 1024^3 B, "
                               f"E0 sweep {E0S[0]}-{E0S[-1]} B, pack+unpack, incount={K} per call",
                   "incount": K,
                   "threads": "hardware_concurrency (PackOptions.threads=0)"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": ncores, "kind": kind,
                         "sample": f"the full step: {K} cfg2 objects per E0, pack + unpack, every E0"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_config_as_gpu_arm": True,
    }
    print(json.dumps(line), flush=True)
    return 0


def build_line(args, value, step_ms, world, K, dominant, sweep, e2e_val, Ke, launches, clk, cpu, halo, send,
               pcie_ms=None, single=None, pattern=None, extra=None):
    hbm, hbm_kind = peaks()
    ms, e0, tag, gbs, li = dominant
    bytes_per_kernel = 2 * K * (1 << 20)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get(f"cfg2_E0_{e0}_{tag}_K{K}")
    # the dominant kernel's physical ceiling: the B200 DRAM transaction rate
    # (HBM peak / 128 B; profiles/r01_dram_granularity.md). Pack of E0 < 128
    # costs one 128-B line read per row; unpack of E0 < 32 a 32-B sector
    # read-modify-write (two transactions) per row.
    if tag == "pack":
        cap = 2 * e0 / (128 + e0) if e0 < 128 else 1.0
    else:
        cap = (e0 / 128 if e0 < 32 else (2 * e0 / (128 + e0) if e0 < 128 else 1.0))
    return {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": f"cfg2: MPI_Type_create_subarray 3D, 1 MiB object in 1024^3 B, "
                               f"E0 sweep {E0S[0]}-{E0S[-1]} B, pack+unpack, incount={K} per call",
                   "incount": K,
                   "l2": "flushed before every timed kernel (512 MiB write, then read back so the timed "
                         "kernel sees a cold clean L2)",
                   "parallelism": f"replicas x{world}"},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(gbs / hbm, 4), "traffic": traffic,
                     "kernel": f"{tag} E0={e0} {li.kernel.name}/w{li.word}",
                     "peak_source": hbm_kind,
                     "algorithmic_bytes_per_launch": bytes_per_kernel,
                     "transaction_cap_frac": round(cap, 4),
                     "frac_of_transaction_cap": round(gbs / hbm / cap, 3),
                     "pattern_cap_GBps": round(pattern, 1) if pattern else None,
                     "frac_of_pattern_cap": round(gbs / pattern, 3) if pattern else None,
                     "pattern_cap_how": "torch strided copy of the same bytes (every 1024th byte of the K GiB "
                                        "allocation), cold L2: the bare DRAM pattern, measured in this run"},
        "sweep": sweep,
        **(extra or {}),
        "single_object": single,
        "e2e": {"value": round(e2e_val, 2), "unit": UNIT, "h2d_bytes_per_step": Ke * (1 << 20) * len(E0S),
                "d2h_bytes_per_step": Ke * (1 << 20) * len(E0S),
                "how": f"sp_pack to / sp_unpack from PINNED HOST message buffers through the C-ABI "
                       f"(the engine pipelines each message over PCIe in 8 MiB chunks: pack kernel + D2H, "
                       f"H2D + unpack kernel); incount={Ke} per E0 message; the packs read one set of "
                       f"objects and the unpacks write another, each E0 on its own pack and unpack stream",
                "issue_order": os.environ.get("BENCH_E2E_ORDER", "ascending") + " E0",
                "pcie_bound_ms": round(pcie_ms, 3) if pcie_ms else None,
                "pcie_bound_note": "the same H2D and D2H bytes as plain pinned copies on two streams at once; "
                                   "e2e ms / this = how far the leg is from the link"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "halo": halo,
        "send": send,
    }


# ------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch
    import ctypes as C

    import paper_2012_14363_b200 as sp
    from paper_2012_14363_b200 import _capi

    rank, local, world = dist_setup(args.gpus)
    # BENCH_DEVICE / BENCH_BACKEND=gloo let several ranks share one GPU in
    # tests (NCCL refuses duplicate devices); the driver uses the defaults
    local = int(os.environ.get("BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("BENCH_BACKEND", "nccl") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K = args.incount
    lib = _capi.lib
    stream = torch.cuda.current_stream()
    sh = C.c_void_p(stream.cuda_stream)

    # one 1024^3 allocation per object: objects one extent (1 GiB) apart
    src = torch.empty((K << 30), dtype=torch.uint8, device="cuda")
    src[::4099] = 3  # touch; content is irrelevant to timing (parity is in tests/)
    packed = torch.zeros(K << 20, dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush_sink = torch.empty((), dtype=torch.int64, device="cuda")

    def flush_l2(i):
        # write 512 MiB (> 126 MB L2), then read it back: the dirty lines are
        # written back during the read, outside the timed window, so the
        # timed kernel starts on a cold, clean L2
        flush.fill_(i & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=flush_sink)

    types = []
    for e0 in E0S:
        d = sp.from_program(cfg2_prog(e0))
        ct = sp.commit_type(d)
        types.append((e0, d, ct))

    pos = C.c_int64(0)

    def call(pack, ct, count, s_ptr, s_len, d_ptr, d_len):
        pos.value = 0
        if pack:
            st = lib.sp_pack(s_ptr, s_len, ct.handle, count, d_ptr, d_len, C.byref(pos), sh)
        else:
            st = lib.sp_unpack(s_ptr, s_len, C.byref(pos), ct.handle, count, d_ptr, d_len, sh)
        if st:
            raise RuntimeError(lib.sp_last_error().decode())

    def one_step(record):
        """pack + unpack of K objects for every E0; returns per-kernel ms"""
        evs = []
        for e0, d, ct in types:
            for pack in (True, False):
                flush_l2(len(evs))
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if pack:
                    call(True, ct, K, src.data_ptr(), src.numel(), packed.data_ptr(), packed.numel())
                else:
                    call(False, ct, K, packed.data_ptr(), packed.numel(), src.data_ptr(), src.numel())
                b.record(stream)
                li = sp.last_launch()
                evs.append((e0, pack, a, b, li))
        return evs

    for _ in range(args.warmup):
        one_step(False)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches0 = sp.kernel_launch_count()
    per = {}  # (e0, pack) -> list of ms
    kinfo = {}
    with ClockSampler(local) as clk:
        all_evs = []
        for _ in range(args.steps):
            all_evs.extend(one_step(True))
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches = sp.kernel_launch_count() - launches0
    for e0, pack, a, b, li in all_evs:
        per.setdefault((e0, pack), []).append(a.elapsed_time(b))
        kinfo[(e0, pack)] = li
    step_ms = sum(sum(v) for v in per.values()) / args.steps
    step_ms = barrier_max(torch, world, step_ms)
    bytes_per_kernel = 2 * K * (1 << 20)
    bytes_per_step = bytes_per_kernel * 2 * len(E0S)
    value = barrier_sum(torch, world, bytes_per_step) / (step_ms * 1e-3) / 1e9
    hbm, hbm_kind = peaks()

    sweep = []
    dominant = None
    for e0 in E0S:
        # caps: 32-B-sector model and the measured B200 DRAM
        # access granularity for isolated rows (128 B per touched line,
        # profiles/r01_dram_granularity.md)
        row = {"E0": e0, "dims": list(cfg2_dims(e0)),
               "sector_cap": round(2 * e0 / (32 + e0), 3) if e0 < 32 else 1.0,
               "line_cap": round(2 * e0 / (128 + e0), 3) if e0 < 128 else 1.0}
        for pack in (True, False):
            ms = statistics.mean(per[(e0, pack)])
            gbs = bytes_per_kernel / (ms * 1e-3) / 1e9
            tag = "pack" if pack else "unpack"
            li = kinfo[(e0, pack)]
            row[f"{tag}_us"] = round(ms * 1e3, 2)
            row[f"{tag}_GBps"] = round(gbs, 1)
            row[f"{tag}_frac"] = round(gbs / hbm, 4)
            row[f"{tag}_kernel"] = f"{li.kernel.name}/w{li.word}"
            if dominant is None or ms > dominant[0]:
                dominant = (ms, e0, tag, gbs, li)
        sweep.append(row)
    # the E0 >= 32 aggregate (the rows the >= 70 %-of-HBM target names):
    # the same bytes-over-time as `value`, restricted to those rows
    big = [e0 for e0 in E0S if e0 >= 32]
    big_ms = sum(statistics.mean(per[(e0, p)]) for e0 in big for p in (True, False))
    value_ge32 = barrier_sum(torch, world, bytes_per_kernel * 2 * len(big)) / (
        barrier_max(torch, world, big_ms) * 1e-3) / 1e9

    # the bare byte pattern of the dominant kernel (outside the timed
    # region): when it is the E0 = 1 pack or unpack, its layout is every
    # 1024th byte of the K GiB allocation, so torch's elementwise strided
    # copy of the same bytes is the same DRAM access pattern with nothing
    # else in the kernel -- the measured cap the kernel is judged against
    pattern = None
    if dominant is not None and dominant[1] == 1:
        strided = src[: (K << 30)].view(-1)[::1024]
        dense = packed[: K << 20]
        ts = []
        for i in range(5):
            flush_l2(i)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if dominant[2] == "unpack":
                strided.copy_(dense)
            else:
                dense.copy_(strided)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        pattern = bytes_per_kernel / (min(ts) * 1e-3) / 1e9
        del strided, dense  # views of src: the e2e leg needs its memory back

    # single objects (outside the timed region): one 1 MiB object per call,
    # the unit the paper reports per pack (cfg1 = vector(131072,1,64,DOUBLE)
    # and every cfg2 E0), cold L2, kernel time by events
    single = []
    for name, prog in [("cfg1", [2, 131072, 1, 64, 0, 3])] + [(f"cfg2 E0={e0}", cfg2_prog(e0)) for e0 in E0S]:
        ct1 = sp.commit_type(sp.from_program(prog))
        r = {"object": name, "bytes": ct1.size}
        for pack in (True, False):
            ts = []
            for i in range(5):
                flush_l2(i)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if pack:
                    call(True, ct1, 1, src.data_ptr(), src.numel(), packed.data_ptr(), packed.numel())
                else:
                    call(False, ct1, 1, packed.data_ptr(), packed.numel(), src.data_ptr(), src.numel())
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            us = min(ts) * 1e3
            tag = "pack" if pack else "unpack"
            r[f"{tag}_us"] = round(us, 2)
            r[f"{tag}_GBps"] = round(2 * ct1.size / us / 1e3, 1)
        single.append(r)
    # what a 1 MiB call costs before any byte moves, under the same flush:
    # two events with nothing between them, a one-thread kernel, and a
    # plain 1 MiB device-to-device copy (a dense copy of the same bytes)
    floors = {}
    tiny = torch.zeros(1, dtype=torch.int32, device="cuda")
    mib_a = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    mib_b = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    for name, fn in (("events_only", lambda: None), ("empty_kernel", lambda: tiny.add_(1)),
                     ("memcpy_1MiB_d2d", lambda: mib_b.copy_(mib_a))):
        ts = []
        for i in range(7):
            flush_l2(i)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        floors[name + "_us"] = round(min(ts) * 1e3, 2)
    single = {"objects": single, "floors": floors,
              "note": "min of 5 (objects) / 7 (floors) cold-L2 calls; a 1 MiB memcpy reads and writes 2 MiB of "
                      "HBM like a 1 MiB pack, so memcpy_1MiB_d2d_us is the floor the pack/unpack times compare to"}
    # cfg1 at the throughput count: 64 vector objects (8-B blocks at 512-B
    # pitch) per call, one extent apart, pack + unpack, cold L2
    ct1 = sp.commit_type(sp.from_program([2, 131072, 1, 64, 0, 3]))
    n1 = min(64, K)  # the packed buffer holds K MiB (--incount below 64)
    cfg1 = {"object": "cfg1 vector(131072,1,64,DOUBLE)", "incount": n1}
    for pack in (True, False):
        ts = []
        for i in range(5):
            flush_l2(i)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if pack:
                call(True, ct1, n1, src.data_ptr(), src.numel(), packed.data_ptr(), packed.numel())
            else:
                call(False, ct1, n1, packed.data_ptr(), packed.numel(), src.data_ptr(), src.numel())
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        li = sp.last_launch()
        ms = statistics.mean(ts)
        tag = "pack" if pack else "unpack"
        gbs = 2 * n1 * ct1.size / (ms * 1e-3) / 1e9
        cfg1[f"{tag}_us"] = round(ms * 1e3, 2)
        cfg1[f"{tag}_GBps"] = round(gbs, 1)
        cfg1[f"{tag}_frac"] = round(gbs / hbm, 4)
        cfg1[f"{tag}_kernel"] = f"{li.kernel.name}/w{li.word}"
    cfg1["line_cap"] = round(2 * 8 / (128 + 8), 4)

    # cfg3 (outside the timed region): the cfg2 object at E0 = 32 built five
    # ways -- subarray, vector of hvector, hvector of vector of hvector,
    # hvector of contiguous, nested subarrays. Every construction must reach
    # the same StridedBlock (so the same kernel and rate); its commit time
    # is reported beside the reference's brute-force commit (SURVEY.md
    # 8(a) T7: 38-103 ms for a cfg2 object).

    e0c, e1c, e2c = 32, 128, 256
    byte = sp.make_named(sp.NamedKind.Byte)
    ways = {
        "subarray": lambda: sp.make_subarray(3, [1024] * 3, [e0c, e1c, e2c], [0, 0, 0], byte),
        "hvector(vector)": lambda: sp.make_hvector(e2c, 1, 1 << 20, sp.make_vector(e1c, e0c, 1024, byte)),
        "hvector(vector(hvector))": lambda: sp.make_hvector(
            e2c, 1, 1 << 20, sp.make_vector(e1c, 1, 1024 // e0c, sp.make_hvector(e0c, 1, 1, byte))),
        "hvector(hvector(contiguous))": lambda: sp.make_hvector(
            e2c, 1, 1 << 20, sp.make_hvector(e1c, 1, 1024, sp.make_contiguous(e0c, byte))),
        "subarray(subarray)": lambda: sp.make_subarray(
            1, [1024], [e2c], [0], sp.make_subarray(2, [1024, 1024], [e0c, e1c], [0, 0], byte)),
    }
    cfg3 = {"object": "cfg2 E0=32 (32 x 128 x 256 B in 1024^3 B)", "incount": K, "rows": []}
    canons = set()
    for name, mk in ways.items():
        tc = []
        for _ in range(20):
            d3 = mk()
            t0 = time.perf_counter()
            c3 = sp.commit_type(d3)
            tc.append(time.perf_counter() - t0)
        canons.add((c3.canon, c3.plan))
        row = {"construction": name, "commit_us": round(statistics.median(tc) * 1e6, 1)}
        for pack in (True, False):
            ts = []
            for i in range(5):
                flush_l2(i)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                if pack:
                    call(True, c3, K, src.data_ptr(), src.numel(), packed.data_ptr(), packed.numel())
                else:
                    call(False, c3, K, packed.data_ptr(), packed.numel(), src.data_ptr(), src.numel())
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            tag = "pack" if pack else "unpack"
            row[f"{tag}_GBps"] = round(2 * K * c3.size / (statistics.median(ts) * 1e-3) / 1e9, 1)
        cfg3["rows"].append(row)
    cfg3["one_canonical_form"] = len(canons) == 1
    cfg3["canon"] = str(next(iter(canons))[0]) if len(canons) == 1 else None

    # e2e: the packed messages live in pinned HOST memory and every call
    # goes through the public C-ABI with those host pointers: sp_pack moves
    # each E0's message out of the device objects to the host (pack kernels,
    # D2H) and sp_unpack moves another message in (H2D, unpack kernels) --
    # the engine pipelines each large message in 8 MiB chunks on a DMA lane
    # beside the caller's stream. The step's packs read one set of objects
    # and its unpacks write a second set, so the two legs are independent
    # (like a halo's sends and receives) and PCIe runs both directions at
    # once: the leg is bounded by the link (pcie_bound_ms). The slow small-E0
    # messages are issued first, so their kernels run while the other
    # messages' bytes are still on the link.
    extra = {"value_E0_ge_32": {"value": round(value_ge32, 2), "unit": UNIT,
                                "frac": round(value_ge32 / hbm, 4),
                                "how": "pack + unpack bytes over kernel time of the E0 >= 32 rows only"},
             "cfg1_throughput": cfg1, "cfg3": cfg3}
    del src, packed
    torch.cuda.empty_cache()
    Ke = min(K, args.e2e_incount)
    NS = int(os.environ.get("BENCH_E2E_STREAMS", len(E0S)))
    xoff, at = {}, 0
    for e0 in sorted(E0S, reverse=True):
        xoff[e0] = at
        at += e0
    esrc = torch.empty((Ke << 30) + 4096, dtype=torch.uint8, device="cuda")  # packed from
    edst = torch.empty((Ke << 30) + 4096, dtype=torch.uint8, device="cuda")  # unpacked into
    msg_in = [torch.full((Ke << 20,), 5, dtype=torch.uint8).pin_memory() for _ in E0S]
    msg_out = [torch.empty(Ke << 20, dtype=torch.uint8).pin_memory() for _ in E0S]
    pstreams = [torch.cuda.Stream() for _ in range(NS)]
    ustreams = [torch.cuda.Stream() for _ in range(NS)]
    phandles = [C.c_void_p(st.cuda_stream) for st in pstreams]
    uhandles = [C.c_void_p(st.cuda_stream) for st in ustreams]
    order = os.environ.get("BENCH_E2E_ORDER", "ascending")
    idx = sorted(range(len(types)), key=lambda i: types[i][0])
    if order == "descending":
        idx = idx[::-1]
    items = [(types[i][2], xoff[types[i][0]], i) for i in idx]  # (type, object offset, E0 index)
    all_streams = pstreams + ustreams
    e2e_t = 0.0
    for it in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(all_streams[0])
        for st in all_streams[1:]:
            st.wait_event(a)
        for n, (ct, off, i) in enumerate(items):
            pos.value = 0
            st = lib.sp_pack(esrc.data_ptr() + off, esrc.numel() - off, ct.handle, Ke, msg_out[i].data_ptr(),
                             msg_out[i].numel(), C.byref(pos), phandles[n % NS])
            assert st == 0, lib.sp_last_error()
            pos.value = 0
            st = lib.sp_unpack(msg_in[i].data_ptr(), msg_in[i].numel(), C.byref(pos), ct.handle, Ke,
                               edst.data_ptr() + off, edst.numel() - off, uhandles[n % NS])
            assert st == 0, lib.sp_last_error()
        for st in all_streams[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            all_streams[0].wait_event(ev)
        b.record(all_streams[0])
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e_t += a.elapsed_time(b)
    streams = all_streams
    # PCIe bound of the leg: the same bytes in both directions at once,
    # plain pinned copies on two streams (no kernels)
    dev_buf = torch.empty(2 * (Ke << 20) * len(E0S), dtype=torch.uint8, device="cuda")
    hin = torch.cat(msg_in).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    half = hin.numel()
    pcie = []
    for it in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        streams[1].wait_event(a)
        with torch.cuda.stream(streams[0]):
            dev_buf[:half].copy_(hin, non_blocking=True)
        with torch.cuda.stream(streams[1]):
            hout.copy_(dev_buf[half:], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(streams[1])
        streams[0].wait_event(ev)
        b.record(streams[0])
        torch.cuda.synchronize()
        if it:
            pcie.append(a.elapsed_time(b))
    pcie_ms = min(pcie)
    del dev_buf, hin, hout
    e2e_ms = barrier_max(torch, world, e2e_t / args.steps)
    e2e_bytes = 2 * Ke * (1 << 20) * 2 * len(E0S)
    e2e_val = barrier_sum(torch, world, e2e_bytes) / (e2e_ms * 1e-3) / 1e9
    del esrc, edst, msg_in, msg_out

    # multi-GPU rows: halo exchange (config 5) and model-selected send (config 4).
    # A watchdog guarantees the driver its JSON line even if these hang.
    del flush
    torch.cuda.empty_cache()
    halo = send = irregular = interpose = None
    line_box = {}
    if not args.no_halo:
        from tools.bench_parts import (halo_section, interpose_section, irregular_section, send_section,
                                       send_self_section)

        def on_timeout():
            if rank == 0 and "line" in line_box:
                line_box["line"]["halo"] = {"error": "timed out"}
                print(json.dumps(line_box["line"]), flush=True)
            os._exit(0)

        cpu_pre = None
        if world == 1 and not args.no_cpu_baseline:  # measured first: the watchdog line needs it
            gbs, t, reps, kind = cpu_sample(1, args.cpu_seconds)
            cpu_pre = {"value": round(gbs, 4), "unit": UNIT, "cores": 1, "kind": kind,
                       "sample": f"{reps} x (pack+unpack of 1 cfg2 object per E0), {t:.1f} s CPU, "
                                 "PackOptions.threads=1 (the reference's fastest setting)"}
            args.no_cpu_baseline = True
            line_box["cpu"] = cpu_pre
        line_box["line"] = build_line(args, value, step_ms, world, K, dominant, sweep, e2e_val, Ke,
                                      launches, clk, cpu_pre, None, None, pcie_ms, single, pattern, extra)
        dog = threading.Timer(args.section_timeout, on_timeout)
        dog.daemon = True
        dog.start()
        job = shared_job_name(world, rank)
        try:
            halo = halo_section(torch, rank, world, local, job)
        except Exception as exc:  # recorded, never fatal to the bench line
            halo = {"error": f"{type(exc).__name__}: {exc}"}
        try:
            if world >= 2:
                send = send_section(torch, rank, world, local, job)
            else:
                send = send_self_section(torch, rank, local, job)
        except Exception as exc:
            send = {"error": f"{type(exc).__name__}: {exc}"}
        try:
            irregular = irregular_section(torch) if rank == 0 else None
        except Exception as exc:
            irregular = {"error": f"{type(exc).__name__}: {exc}"}
        try:  # the drop-in over a system MPI: same binary with / without the interposer
            interpose = interpose_section() if world == 1 and not args.no_interpose else None
        except Exception as exc:
            interpose = {"error": f"{type(exc).__name__}: {exc}"}
        dog.cancel()

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0
    cpu = line_box.get("cpu")
    if cpu is None and world == 1 and not args.no_cpu_baseline:
        gbs, t, reps, kind = cpu_sample(1, args.cpu_seconds)
        cpu = {"value": round(gbs, 4), "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"{reps} x (pack+unpack of 1 cfg2 object per E0), {t:.1f} s CPU, "
                         "PackOptions.threads=1 (the reference's fastest setting)"}
    line = build_line(args, value, step_ms, world, K, dominant, sweep, e2e_val, Ke, launches, clk, cpu, halo,
                      send, pcie_ms, single, pattern, extra)
    line["irregular_types"] = irregular
    line["interpose"] = interpose
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--incount", type=int, default=64)
    ap.add_argument("--e2e-incount", type=int, default=64)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-halo", action="store_true", help="skip the halo / send sections")
    ap.add_argument("--no-interpose", action="store_true",
                    help="skip the interposer-over-a-system-MPI section (N=1 only)")
    ap.add_argument("--section-timeout", type=float, default=420.0,
                    help="watchdog (s) for the halo/send sections; the bench line is printed regardless")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

// model.cpp -- send-method model (paper Eqs. 1-3) over a machine profile.
//
// Semantics follow perf_model.hpp:17-229 and profile_io.hpp:88-213 of the
// reference (log-log piecewise-linear 1D curves, log-log bilinear 2D
// surfaces clamped at the edges, argmin with device > one-shot > staged
// ties, the line-oriented text format); the profile this engine ships is
// MEASURED on B200 by tools/measure (profiles/b200.profile).
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <shared_mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "core.hpp"
#include "model.hpp"

namespace spb {

// ------------------------------------------------------------ interpolation
namespace {

struct Pos {
  size_t lo, hi;
  double u; // log-space position in [lo, hi]
};

// clamp outside the sampled range, exact on knots (perf_model.hpp:75-97)
Pos locate(const std::vector<double> &xs, double q) {
  const size_t n = xs.size();
  if (q <= xs[0]) return {0, 0, 0.0};
  if (q >= xs[n - 1]) return {n - 1, n - 1, 0.0};
  size_t hi = 1;
  while (xs[hi] < q) ++hi;
  if (xs[hi] == q) return {hi, hi, 0.0};
  const size_t lo = hi - 1;
  if (xs[lo] == q) return {lo, lo, 0.0};
  return {lo, hi, (std::log(q) - std::log(xs[lo])) / (std::log(xs[hi]) - std::log(xs[lo]))};
}

// geometric blend; arithmetic when a sample is zero (perf_model.hpp:100-108)
double blend(double a, double b, double u) {
  if (a == b) return a;
  if (a <= 0.0 || b <= 0.0) return (1.0 - u) * a + u * b;
  return std::exp((1.0 - u) * std::log(a) + u * std::log(b));
}

} // namespace

double interp_1d(const Curve &c, double x) {
  if (c.size.empty()) fail(SP_ERR_EMPTY_PROFILE, "interp_1d: curve has no samples");
  const Pos p = locate(c.size, x);
  return p.lo == p.hi ? c.time[p.lo] : blend(c.time[p.lo], c.time[p.hi], p.u);
}

double interp_2d(const Surface &s, double obj, double blk) {
  if (s.object.empty() || s.block.empty()) fail(SP_ERR_EMPTY_PROFILE, "interp_2d: surface has no samples");
  const Pos po = locate(s.object, obj), pb = locate(s.block, blk);
  const size_t nb = s.block.size();
  auto at = [&](size_t i, size_t j) { return s.time[i * nb + j]; };
  const double t0 = blend(at(po.lo, pb.lo), at(po.hi, pb.lo), po.u);
  const double t1 = blend(at(po.lo, pb.hi), at(po.hi, pb.hi), po.u);
  return blend(t0, t1, pb.u);
}

ModelTimes model_times(const Profile &p, int64_t object_size, int64_t block_size) {
  const double o = static_cast<double>(object_size), b = static_cast<double>(block_size);
  ModelTimes t;
  // Eq. 1 device  = gpu_pack + gpu_gpu + gpu_unpack
  t.device = interp_2d(p.surf[SP_SURF_GPU_PACK], o, b) + interp_1d(p.curve[SP_CURVE_GPU_GPU], o) +
             interp_2d(p.surf[SP_SURF_GPU_UNPACK], o, b);
  // Eq. 2 oneshot = host_pack + cpu_cpu + host_unpack
  t.oneshot = interp_2d(p.surf[SP_SURF_HOST_PACK], o, b) + interp_1d(p.curve[SP_CURVE_CPU_CPU], o) +
              interp_2d(p.surf[SP_SURF_HOST_UNPACK], o, b);
  // Eq. 3 staged  = gpu_pack + d2h + cpu_cpu + h2d + gpu_unpack
  t.staged = interp_2d(p.surf[SP_SURF_GPU_PACK], o, b) + interp_1d(p.curve[SP_CURVE_D2H], o) +
             interp_1d(p.curve[SP_CURVE_CPU_CPU], o) + interp_1d(p.curve[SP_CURVE_H2D], o) +
             interp_2d(p.surf[SP_SURF_GPU_UNPACK], o, b);
  return t;
}

int choose_method(const Profile &p, int64_t object_size, int64_t block_size) {
  if (object_size <= 0 || block_size <= 0 || block_size > object_size)
    fail(SP_ERR_INVALID_ARGUMENT, "choose_method: need 0 < block_size <= object_size");
  const ModelTimes t = model_times(p, object_size, block_size);
  // ties prefer fewer hops (perf_model.hpp:169-178)
  int best = SP_METHOD_DEVICE;
  double bt = t.device;
  if (t.oneshot < bt) {
    best = SP_METHOD_ONESHOT;
    bt = t.oneshot;
  }
  if (t.staged < bt) best = SP_METHOD_STAGED;
  return best;
}

int choose_method_b200(const Profile &p, int64_t object_size, int64_t block_size, int dst_kind, double times[4]) {
  const int ref = choose_method(p, object_size, block_size);
  const ModelTimes t = model_times(p, object_size, block_size);
  const Surface *direct = dst_kind == kDstSameGpu   ? &p.surf[SP_SURF_GPU_DIRECT]
                          : dst_kind == kDstPeerGpu ? &p.surf[SP_SURF_GPU_DIRECT_PEER]
                                                    : nullptr;
  const double td = direct && !direct->object.empty()
                        ? interp_2d(*direct, static_cast<double>(object_size), static_cast<double>(block_size))
                        : HUGE_VAL;
  if (times) {
    times[0] = t.device;
    times[1] = t.oneshot;
    times[2] = t.staged;
    times[3] = td;
  }
  const double tref = ref == SP_METHOD_DEVICE ? t.device : ref == SP_METHOD_ONESHOT ? t.oneshot : t.staged;
  return td <= tref ? SP_METHOD_DIRECT : ref;
}

// ------------------------------------------------------------ text format
namespace {

const char *kCurveNames[4] = {"cpu_cpu", "gpu_gpu", "d2h", "h2d"};
const char *kSurfNames[6] = {"gpu_pack", "gpu_unpack", "host_pack", "host_unpack", "gpu_direct", "gpu_direct_peer"};

template <int N> int name_index(const char *const (&names)[N], const std::string &s) {
  for (int i = 0; i < N; ++i)
    if (s == names[i]) return i;
  return -1;
}

[[noreturn]] void parse_fail(int line, const std::string &m) {
  fail(SP_ERR_PARSE, "profile line " + std::to_string(line) + ": " + m);
}

void check_curve(const Curve &c, const char *name) {
  for (size_t i = 0; i < c.size.size(); ++i) {
    if (c.size[i] <= 0 || c.time[i] < 0)
      fail(SP_ERR_PARSE, std::string("profile: curve ") + name + " needs positive sizes and nonnegative times");
    if (i && c.size[i] <= c.size[i - 1])
      fail(SP_ERR_PARSE, std::string("profile: curve ") + name + " sizes must be strictly increasing");
  }
}

// rows in any order -> complete rectangular grid (profile_io.hpp:42-78)
Surface grid_of(const std::vector<std::array<double, 3>> &rows, const char *name) {
  std::map<double, size_t> ox, bx;
  for (const auto &r : rows) {
    if (r[0] <= 0 || r[1] <= 0 || r[2] < 0)
      fail(SP_ERR_PARSE, std::string("profile: surface ") + name + " needs positive sizes and nonnegative times");
    ox.emplace(r[0], 0);
    bx.emplace(r[1], 0);
  }
  Surface s;
  for (auto &kv : ox) {
    kv.second = s.object.size();
    s.object.push_back(kv.first);
  }
  for (auto &kv : bx) {
    kv.second = s.block.size();
    s.block.push_back(kv.first);
  }
  if (rows.size() != ox.size() * bx.size())
    fail(SP_ERR_PARSE, std::string("profile: surface ") + name + " grid is incomplete or has duplicate points");
  s.time.assign(ox.size() * bx.size(), -1.0);
  for (const auto &r : rows) {
    double &cell = s.time[ox[r[0]] * bx.size() + bx[r[1]]];
    if (cell >= 0) fail(SP_ERR_PARSE, std::string("profile: surface ") + name + " has duplicate points");
    cell = r[2];
  }
  return s;
}

} // namespace

Profile parse_profile(const std::string &text) {
  Profile p;
  std::vector<std::array<double, 3>> rows[6];
  bool have_rows[6] = {false, false, false, false, false, false};
  int cur_curve = -1, cur_surf = -1;
  std::istringstream in(text);
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const auto hash = line.find('#');
    std::istringstream ls(hash == std::string::npos ? line : line.substr(0, hash));
    std::string first;
    if (!(ls >> first)) continue;
    if (first == "curve") {
      std::string nm;
      if (!(ls >> nm) || (cur_curve = name_index(kCurveNames, nm)) < 0) parse_fail(lineno, "unknown curve name");
      cur_surf = -1;
    } else if (first == "surface") {
      std::string nm;
      if (!(ls >> nm) || (cur_surf = name_index(kSurfNames, nm)) < 0) parse_fail(lineno, "unknown surface name");
      have_rows[cur_surf] = true;
      cur_curve = -1;
    } else {
      char *end = nullptr;
      const double a = std::strtod(first.c_str(), &end);
      if (end == first.c_str() || *end != '\0') parse_fail(lineno, "expected a number, got '" + first + "'");
      if (cur_curve >= 0) {
        double t;
        if (!(ls >> t)) parse_fail(lineno, "curve rows are `size_bytes time_seconds`");
        p.curve[cur_curve].size.push_back(a);
        p.curve[cur_curve].time.push_back(t);
      } else if (cur_surf >= 0) {
        double b, t;
        if (!(ls >> b >> t)) parse_fail(lineno, "surface rows are `object_bytes block_bytes time_seconds`");
        rows[cur_surf].push_back({a, b, t});
      } else {
        parse_fail(lineno, "data row before any section header");
      }
    }
  }
  // curves are validated in name order (the reference iterates a std::map)
  for (int i : {SP_CURVE_CPU_CPU, SP_CURVE_D2H, SP_CURVE_GPU_GPU, SP_CURVE_H2D}) check_curve(p.curve[i], kCurveNames[i]);
  for (int i : {SP_SURF_GPU_PACK, SP_SURF_GPU_UNPACK, SP_SURF_HOST_PACK, SP_SURF_HOST_UNPACK, SP_SURF_GPU_DIRECT,
                SP_SURF_GPU_DIRECT_PEER})
    if (have_rows[i]) p.surf[i] = grid_of(rows[i], kSurfNames[i]);
  return p;
}

std::string format_profile(const Profile &p, const std::string &header) {
  std::string out;
  char buf[64];
  auto num = [&](double v) {
    std::snprintf(buf, sizeof buf, "%.9e", v);
    return std::string(buf);
  };
  if (!header.empty()) {
    std::istringstream hs(header);
    std::string h;
    while (std::getline(hs, h)) out += "# " + h + "\n";
  }
  for (int i = 0; i < 4; ++i) {
    out += std::string("curve ") + kCurveNames[i] + "\n";
    for (size_t k = 0; k < p.curve[i].size.size(); ++k)
      out += num(p.curve[i].size[k]) + " " + num(p.curve[i].time[k]) + "\n";
  }
  for (int i = 0; i < 6; ++i) {
    const Surface &s = p.surf[i];
    if (i >= 4 && s.object.empty()) continue; // extension surfaces only when measured
    out += std::string("surface ") + kSurfNames[i] + "\n";
    for (size_t a = 0; a < s.object.size(); ++a)
      for (size_t b = 0; b < s.block.size(); ++b)
        out += num(s.object[a]) + " " + num(s.block[b]) + " " + num(s.time[a * s.block.size() + b]) + "\n";
  }
  return out;
}

// ------------------------------------------------------------ cache
// Memoised choose_method keyed on (object, block). 32 shards, each a hash
// map under its own reader/writer lock; a miss computes outside the lock.
// Lock-free on the hit path: a direct-mapped table of 2^16 slots, each two
// atomic words (object size; block size << 3 | method << 1 | valid). A
// reader loads tag, object, tag again and accepts only an unchanged, valid
// tag whose object and block match -- a concurrent writer can only cause a
// miss, and a miss recomputes choose_method, so answers are always exact.
// Colliding queries overwrite each other (it is a cache of a pure function).
struct ModelCache {
  explicit ModelCache(std::shared_ptr<const Profile> p) : prof(std::move(p)), sets(new Set[kSets]) {}
  static constexpr size_t kSets = size_t{1} << 14; // x 4 ways = 64 Ki entries, 1 MiB
  struct Slot {
    std::atomic<uint64_t> tag{0};
    std::atomic<uint64_t> obj{0};
  };
  struct alignas(64) Set {
    Slot way[4];
  };
  std::shared_ptr<const Profile> prof;
  std::unique_ptr<Set[]> sets;

  static uint64_t hash(int64_t o, int64_t b) {
    uint64_t h = static_cast<uint64_t>(o) * 0xd6e8feb86659fd93ull ^ static_cast<uint64_t>(b);
    h ^= h >> 31;
    h *= 0x9e3779b97f4a7c15ull;
    return h ^ (h >> 29);
  }

  static constexpr uint64_t kBusy = 2; // invalid (bit 0 clear), nonzero: a writer owns the slot

  int choose(int64_t o, int64_t b) {
    const uint64_t h = hash(o, b);
    Set &set = sets[h & (kSets - 1)];
    for (Slot &s : set.way) {
      const uint64_t t1 = s.tag.load(std::memory_order_acquire);
      const uint64_t ob = s.obj.load(std::memory_order_acquire);
      const uint64_t t2 = s.tag.load(std::memory_order_acquire);
      if (t1 == t2 && (t1 & 1) && ob == static_cast<uint64_t>(o) && (t1 >> 3) == static_cast<uint64_t>(b))
        return static_cast<int>((t1 >> 1) & 3);
    }
    const int m = choose_method(*prof, o, b);
    if (b >= 0 && b < (int64_t{1} << 60)) { // publish: invalidate, write, validate
      Slot *victim = &set.way[(h >> 40) & 3];
      for (Slot &s : set.way)
        if (!(s.tag.load(std::memory_order_relaxed) & 1)) {
          victim = &s;
          break;
        }
      // claim the slot (valid or empty -> busy) so that two writers never
      // interleave their obj and tag stores; a slot another thread is
      // filling is left to it (this answer is simply not cached)
      uint64_t cur = victim->tag.load(std::memory_order_relaxed);
      if (cur != kBusy && victim->tag.compare_exchange_strong(cur, kBusy, std::memory_order_acq_rel)) {
        victim->obj.store(static_cast<uint64_t>(o), std::memory_order_release);
        victim->tag.store(static_cast<uint64_t>(b) << 3 | static_cast<uint64_t>(m) << 1 | 1,
                          std::memory_order_release);
      }
    }
    return m;
  }
};

} // namespace spb

// ============================================================ C-ABI
using spb::Profile;

struct sp_model_cache_s {
  spb::ModelCache c;
};

namespace {
template <class F> sp_status guard_m(F &&f) {
  try {
    spb::set_last_error("");
    f();
    return SP_OK;
  } catch (const spb::Error &e) {
    spb::set_last_error(e.msg);
    return e.code;
  } catch (const std::exception &e) {
    spb::set_last_error(e.what());
    return SP_ERR_INTERNAL;
  }
}
void need(const void *p) {
  if (!p) spb::fail(SP_ERR_INVALID_ARGUMENT, "null argument");
}
} // namespace

extern "C" {

sp_status sp_profile_create(sp_profile *out) {
  return guard_m([&] {
    need(out);
    *out = new sp_profile_s{std::make_shared<Profile>()};
  });
}

sp_status sp_profile_parse(const char *text, sp_profile *out) {
  return guard_m([&] {
    need(text);
    need(out);
    *out = new sp_profile_s{std::make_shared<Profile>(spb::parse_profile(text))};
  });
}

sp_status sp_profile_load(const char *path, sp_profile *out) {
  return guard_m([&] {
    need(path);
    need(out);
    std::ifstream in(path);
    if (!in) spb::fail(SP_ERR_PARSE, std::string("cannot open profile file: ") + path);
    std::stringstream ss;
    ss << in.rdbuf();
    *out = new sp_profile_s{std::make_shared<Profile>(spb::parse_profile(ss.str()))};
  });
}

sp_status sp_profile_save(sp_profile p, const char *header, char *buf, int64_t cap, int64_t *len) {
  return guard_m([&] {
    need(p);
    need(len);
    const std::string s = spb::format_profile(*p->p, header ? header : "");
    *len = static_cast<int64_t>(s.size());
    if (buf && cap > *len) {
      std::memcpy(buf, s.data(), s.size());
      buf[s.size()] = 0;
    } else if (buf) {
      spb::fail(SP_ERR_BUFFER_TOO_SMALL, "profile text needs " + std::to_string(s.size() + 1) + " bytes");
    }
  });
}

sp_status sp_profile_free(sp_profile p) {
  delete p;
  return SP_OK;
}

sp_status sp_profile_set_curve(sp_profile p, int curve, const double *size, const double *time, int64_t n) {
  return guard_m([&] {
    need(p);
    if (curve < 0 || curve > 3 || n < 0) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad curve");
    spb::Curve c;
    c.size.assign(size, size + n);
    c.time.assign(time, time + n);
    p->p->curve[curve] = std::move(c);
  });
}

sp_status sp_profile_set_surface(sp_profile p, int surf, const double *object, int64_t nobj, const double *block,
                                 int64_t nblk, const double *time) {
  return guard_m([&] {
    need(p);
    if (surf < 0 || surf > 5 || nobj < 0 || nblk < 0) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad surface");
    spb::Surface s;
    s.object.assign(object, object + nobj);
    s.block.assign(block, block + nblk);
    s.time.assign(time, time + nobj * nblk);
    p->p->surf[surf] = std::move(s);
  });
}

sp_status sp_interp_1d(sp_profile p, int curve, double size, double *t) {
  return guard_m([&] {
    need(p);
    need(t);
    if (curve < 0 || curve > 3) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad curve");
    *t = spb::interp_1d(p->p->curve[curve], size);
  });
}

sp_status sp_interp_2d(sp_profile p, int surf, double object, double block, double *t) {
  return guard_m([&] {
    need(p);
    need(t);
    if (surf < 0 || surf > 5) spb::fail(SP_ERR_INVALID_ARGUMENT, "bad surface");
    *t = spb::interp_2d(p->p->surf[surf], object, block);
  });
}

sp_status sp_model_times(sp_profile p, int64_t object_size, int64_t block_size, double *t_device,
                         double *t_oneshot, double *t_staged) {
  return guard_m([&] {
    need(p);
    const spb::ModelTimes t = spb::model_times(*p->p, object_size, block_size);
    if (t_device) *t_device = t.device;
    if (t_oneshot) *t_oneshot = t.oneshot;
    if (t_staged) *t_staged = t.staged;
  });
}

sp_status sp_choose_method(sp_profile p, int64_t object_size, int64_t block_size, int *method) {
  return guard_m([&] {
    need(p);
    need(method);
    *method = spb::choose_method(*p->p, object_size, block_size);
  });
}

sp_status sp_choose_method_b200(sp_profile p, int64_t object_size, int64_t block_size, int dst_kind, int *method,
                                double times[4]) {
  return guard_m([&] {
    need(p);
    need(method);
    if (dst_kind < 0 || dst_kind > 2) spb::fail(SP_ERR_INVALID_ARGUMENT, "dst_kind must be 0, 1 or 2");
    *method = spb::choose_method_b200(*p->p, object_size, block_size, dst_kind, times);
  });
}

sp_status sp_model_cache_create(sp_profile p, sp_model_cache *out) {
  return guard_m([&] {
    need(p);
    need(out);
    *out = new sp_model_cache_s{spb::ModelCache(p->p)};
  });
}

sp_status sp_model_cache_choose(sp_model_cache c, int64_t object_size, int64_t block_size, int *method) {
  return guard_m([&] {
    need(c);
    need(method);
    *method = c->c.choose(object_size, block_size);
  });
}

sp_status sp_model_cache_free(sp_model_cache c) {
  delete c;
  return SP_OK;
}

} // extern "C"

// model.hpp -- machine profile + send-method model (internal).
#pragma once

#include <string>
#include <vector>

#include "stridepack_b200.h"

namespace spb {

struct Curve {            // transfer time vs bytes (perf_model.hpp:17-21)
  std::vector<double> size, time;
};
struct Surface {          // pack time vs (object, block) (perf_model.hpp:24-28)
  std::vector<double> object, block;
  std::vector<double> time; // row-major [object][block]
};
struct Profile {          // MachineProfile (perf_model.hpp:36-45)
  Curve curve[4];         // SP_CURVE_*
  // SP_SURF_*: the reference's four, then the B200 extension's optional
  // DIRECT surfaces (one typed-copy launch source layout -> destination
  // layout, same GPU / into a peer GPU over NVLink); empty when unmeasured
  Surface surf[6];
};
struct ModelTimes {
  double device, oneshot, staged;
};

// Destination of a message, for the B200 method choice.
enum DstKind { kDstHost = 0, kDstSameGpu = 1, kDstPeerGpu = 2 };

double interp_1d(const Curve &c, double x);
double interp_2d(const Surface &s, double obj, double blk);
ModelTimes model_times(const Profile &p, int64_t object_size, int64_t block_size);
int choose_method(const Profile &p, int64_t object_size, int64_t block_size);
// B200 extension: Eqs. 1-3 plus Eq. 4, t_direct = the DIRECT surface of the
// destination (same GPU or peer GPU); DIRECT competes only for device
// destinations whose surface was measured. times[4] = device, one-shot,
// staged, direct (+inf when not a candidate). Ties prefer DIRECT (one
// launch, no intermediate), then the reference's order.
int choose_method_b200(const Profile &p, int64_t object_size, int64_t block_size, int dst_kind, double times[4]);
Profile parse_profile(const std::string &text);
std::string format_profile(const Profile &p, const std::string &header);

} // namespace spb

struct sp_profile_s {     // the C-ABI handle
  std::shared_ptr<spb::Profile> p;
};

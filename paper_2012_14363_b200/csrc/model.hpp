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
  Surface surf[4];        // SP_SURF_*
};
struct ModelTimes {
  double device, oneshot, staged;
};

double interp_1d(const Curve &c, double x);
double interp_2d(const Surface &s, double obj, double blk);
ModelTimes model_times(const Profile &p, int64_t object_size, int64_t block_size);
int choose_method(const Profile &p, int64_t object_size, int64_t block_size);
Profile parse_profile(const std::string &text);
std::string format_profile(const Profile &p, const std::string &header);

} // namespace spb

struct sp_profile_s {     // the C-ABI handle
  std::shared_ptr<spb::Profile> p;
};

// tools/measure_profile.cpp -- measure this B200 node and write a machine
// profile in the reference's format (profile_io.hpp:174-213). Replaces the
// reference's profile-gen (cli.hpp:177-233), which timed its host executor
// and left every transfer curve synthetic. Native C++ over the C-ABI, so the
// samples are the latencies the engine's own send paths see:
//
//   gpu_pack / gpu_unpack    sp_pack / sp_unpack, device <-> device
//   host_pack / host_unpack  one-shot kernels: pack into / unpack from
//                            pinned, mapped host memory
//   gpu_gpu                  packed bytes GPU -> GPU: cudaMemcpyPeerAsync to
//                            device 1 when visible, else same-device copy
//   d2h / h2d                cudaMemcpyAsync to / from pinned host memory
//   cpu_cpu                  pinned host memcpy (the node-local runtime shares
//                            host regions; one copy stands in for the wire)
//
// Each sample: median of `reps` synchronous calls (enqueue + completion).
// Surfaces probe hvector(o/b, 1, 2b, contiguous(b, BYTE)) like profile-gen.
//
//   measure_profile <out.profile> [reps]
#include <cstdlib>

#include "measure.hpp"

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s out.profile [reps]\n", argv[0]);
    return 2;
  }
  return measure_profile(argv[1], argc > 2 ? std::atoi(argv[2]) : 25, true);
}

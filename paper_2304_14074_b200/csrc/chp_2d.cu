// 2D propagators (configs 3-5) -- placeholder until the DST/PCG kernels land.
#include <string>

#include "chp_common.cuh"

struct Chp2d {};
Chp2d* chp2d_create() { return new Chp2d(); }
void chp2d_destroy(Chp2d* c) { delete c; }

cudaError_t chp2d_propagate(Chp2d*, const chp_grid&, const chp_spec&, int, int, const double*,
                            long long, double*, long long, const int*, chp_sys_info*,
                            cudaStream_t, std::string* err) {
  *err = "2D propagators not built yet";
  return cudaSuccess;
}
cudaError_t chp2d_coarse_sweep(Chp2d*, const chp_grid&, const chp_spec&, int, int, int, int, int,
                               double*, const double*, double*, long long, long long,
                               unsigned char*, double*, chp_sys_info*, cudaStream_t,
                               std::string* err) {
  *err = "2D coarse sweep not built yet";
  return cudaSuccess;
}

// Shared device helpers for the chparareal B200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/chp.h"

#define CHP_DEV __device__ __forceinline__

// ---------------------------------------------------------------------------
// v^3 with a fixed IEEE operation sequence (bit-identical to
// oracle/chp_oracle.py:exact_cube): p+e = v*v and P+E = p*v are exact
// two-products, result = P + (E + e*v).  Every op is an explicit _rn
// intrinsic so the compiler cannot contract or reorder.
// ---------------------------------------------------------------------------
CHP_DEV double chp_cube(double v) {
  const double p = __dmul_rn(v, v);
  const double e = __fma_rn(v, v, -p);
  const double P = __dmul_rn(p, v);
  const double E = __fma_rn(p, v, -P);
  return __dadd_rn(P, __dadd_rn(E, __dmul_rn(e, v)));
}

// w = v^3 - 3v  (schemes.py:260: v**3 - 3.0*v)
CHP_DEV double chp_cube_minus_3v(double v) {
  return __dsub_rn(chp_cube(v), __dmul_rn(3.0, v));
}

// Per-system result record shared by every propagate / sweep kernel.
struct SysInfo {
  int status;          // chp_sys_status
  int fail_iter;       // Newton iteration count at failure
  double fail_resid;   // residual at failure
  long long newton_steps;
  long long newton_total;
  int newton_max;
  int cg_max;          // max CG iterations seen (2D)
  double newton_maxres;
  long long cg_total;  // total CG iterations (2D)
};
static_assert(sizeof(SysInfo) == sizeof(chp_sys_info), "SysInfo layout");

CHP_DEV void sysinfo_fail(SysInfo* si, int status, int it, double r) {
  if (si->status == CHP_SYS_OK) {
    si->status = status;
    si->fail_iter = it;
    si->fail_resid = r;
  }
}

// max of non-negative doubles via the ordered int64 bit pattern (order
// independent -> deterministic)
CHP_DEV void atomic_max_nonneg(double* addr, double v) {
  if (!(v >= 0.0)) v = __longlong_as_double(0x7ff0000000000000LL);  // NaN -> +inf
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

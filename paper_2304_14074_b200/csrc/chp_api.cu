#include <cuda.h>
#include <string.h>
// C ABI of libchp.so (include/chp.h): context, caches, dispatch.
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "chp_common.cuh"

// launchers defined in chp_1d.cu / chp_2d.cu / chp_engine.cu
cudaError_t chp1d_factor(const chp_grid& g, double dt, double b, double* fac, int* err,
                         cudaStream_t st);
cudaError_t chp1d_propagate(const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                            const double* in, long long in_stride, double* out,
                            long long out_stride, const int* sys_index, const double* fac,
                            double* ub, double* yh, double* tmp, chp_sys_info* info,
                            cudaStream_t st, double* hist, int hlen);
cudaError_t chp1d_coarse_sweep(const chp_grid& g, const chp_spec& sp, int mode, int nic, int nsl,
                               int n0, int n1, double* U, const double* F, double* G,
                               long long ic_stride, long long sl_stride, unsigned char* changed,
                               double* inc, const double* fac, double* ub, double* yh,
                               double* tmp, chp_sys_info* info, cudaStream_t st);
cudaError_t chp_launch_max_abs_diff(const chp_grid& g, int n_fields, const double* a,
                                    long long as, const double* b, long long bs, double* out,
                                    cudaStream_t st);
cudaError_t chp_launch_field_stats(const chp_grid& g, int n_fields, const double* in,
                                   long long stride, double* out, cudaStream_t st);
cudaError_t chp_launch_dfma_probe(int blocks, int iters, double* out, cudaStream_t st);
size_t chp_nn_scratch_bytes(int step, int nsys, int S);
cudaError_t chp_nn_launch(const chp_grid& gr, const chp_nn_params& p, double dt, double eps2,
                          int steps, int nsys, const double* in, long long in_stride,
                          double* out, long long out_stride, const int* sys_index,
                          const double* traces_in, double* traces_out, chp_sys_info* info,
                          double* scratch, cudaStream_t st);
struct Chp2d;
Chp2d* chp2d_create();
void chp2d_destroy(Chp2d*);
cudaError_t chp2d_propagate(Chp2d* c, const chp_grid& g, const chp_spec& sp, int steps, int nsys,
                            const double* in, long long in_stride, double* out,
                            long long out_stride, const int* sys_index, chp_sys_info* info,
                            double* hist, int hlen, cudaStream_t st, std::string* err);
cudaError_t chp2d_coarse_sweep(Chp2d* c, const chp_grid& g, const chp_spec& sp, int mode,
                               int nic, int nsl, int n0, int n1, double* U, const double* F,
                               double* G, long long ic_stride, long long sl_stride,
                               unsigned char* changed, double* inc, chp_sys_info* info,
                               cudaStream_t st, std::string* err, const chp_hop* hop, bool* fused);
cudaError_t chp_launch_hop_put(long long fs, int nic, const double* src, long long src_stride,
                               const unsigned char* changed, long long changed_stride,
                               const chp_hop& hop, cudaStream_t st);
cudaError_t chp_launch_hop_take(long long fs, int nic, const double* mail, long long mail_stride,
                                const unsigned char* mail_changed, double* U0, long long ic_stride,
                                unsigned char* changed, long long changed_stride,
                                unsigned int* peer_ack, unsigned int seq, cudaStream_t st);

struct chp_ctx {
  int device = 0;
  std::string last_error;
  // cached 1D Cholesky factors keyed by (m, c1, dt, b) -- _FACTOR_CACHE analogue
  std::map<std::tuple<int, double, double, double>, double*> factors;
  // grow-only 1D scratch
  double* scratch = nullptr;
  size_t scratch_bytes = 0;
  int* dev_err = nullptr;
  Chp2d* d2 = nullptr;
  // every entry point holds the lock from argument checks through the launches:
  // the factor map, scratch, 2D workspaces and last_error are shared state (the
  // reference calls propagate from worker threads)
  std::mutex mu;
};

// Switch to the context's device for the duration of an entry point and restore
// the caller's current device afterwards (kernels, caches and scratch all live on
// ctx->device whatever device the caller has current).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

namespace {

chp_status fail(chp_ctx* c, chp_status s, const std::string& msg) {
  if (c) c->last_error = msg;
  return s;
}

chp_status cuda_fail(chp_ctx* c, cudaError_t e, const char* where) {
  return fail(c, CHP_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool grid_ok(const chp_grid* g, std::string* why) {
  if (!g) { *why = "null grid"; return false; }
  if (g->dim != 1 && g->dim != 2) { *why = "dim must be 1 or 2"; return false; }
  if (g->nx < 4) { *why = "nodes_per_axis must be at least 4"; return false; }
  if (g->m != g->nx - 2) { *why = "m must equal nx - 2"; return false; }
  if (g->pitch < g->m) { *why = "pitch must be >= m"; return false; }
  return true;
}

bool spec_ok(const chp_spec* s, std::string* why) {
  if (!s) { *why = "null spec"; return false; }
  if (s->scheme < CHP_LINEAR_A || s->scheme > CHP_NONLINEAR_EYRE) {
    *why = "unknown scheme";
    return false;
  }
  if (!(s->dt > 0)) { *why = "dt must be positive"; return false; }
  if (!(s->eps > 0)) { *why = "eps must be positive"; return false; }
  if (!(s->newton_tol > 0)) { *why = "newton_tol must be positive"; return false; }
  if (s->newton_max_iter < 1) { *why = "newton_max_iter must be at least 1"; return false; }
  return true;
}

// Scratch for the 1D kernels: ub [m][6][n] + yh [m][n] + tmp [m][n].
chp_status ensure_scratch(chp_ctx* c, size_t bytes, cudaStream_t st) {
  if (bytes <= c->scratch_bytes) return CHP_OK;
  if (c->scratch) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(c, e, "sync before scratch grow");
    cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&c->scratch, bytes);
  if (e != cudaSuccess) return cuda_fail(c, e, "scratch alloc");
  c->scratch_bytes = bytes;
  return CHP_OK;
}

chp_status factor_1d(chp_ctx* c, const chp_grid* g, double dt, double b, cudaStream_t st,
                     const double** out) {
  auto key = std::make_tuple(g->m, g->c1, dt, b);
  auto it = c->factors.find(key);
  if (it != c->factors.end()) { *out = it->second; return CHP_OK; }
  double* fac = nullptr;
  cudaError_t e = cudaMalloc(&fac, sizeof(double) * 4 * g->m);
  if (e != cudaSuccess) return cuda_fail(c, e, "factor alloc");
  e = chp1d_factor(*g, dt, b, fac, c->dev_err, st);
  if (e != cudaSuccess) { cudaFree(fac); return cuda_fail(c, e, "factor launch"); }
  int herr = 0;
  e = cudaMemcpyAsync(&herr, c->dev_err, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { cudaFree(fac); return cuda_fail(c, e, "factor sync"); }
  if (herr != 0) {
    cudaFree(fac);
    char buf[128];
    snprintf(buf, sizeof buf, "%d-th leading minor not positive definite", herr);
    return fail(c, CHP_ERR_ARG, buf);
  }
  c->factors[key] = fac;
  *out = fac;
  return CHP_OK;
}

}  // namespace

extern "C" {

const char* chp_version(void) { return "chp-b200 0.1 (sm_100a)"; }

const char* chp_status_str(int s) {
  switch (s) {
    case CHP_OK: return "ok";
    case CHP_ERR_ARG: return "invalid argument";
    case CHP_ERR_CUDA: return "cuda error";
    case CHP_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}

chp_status chp_ctx_create(int device, chp_ctx** out) {
  if (!out) return CHP_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return CHP_ERR_CUDA;
  DeviceGuard dg(device);
  cudaError_t e = cudaSuccess;
  chp_ctx* c = new chp_ctx();
  c->device = device;
  e = cudaMalloc(&c->dev_err, sizeof(int) * 4);
  if (e != cudaSuccess) { delete c; return CHP_ERR_CUDA; }
  c->d2 = chp2d_create();
  *out = c;
  return CHP_OK;
}

chp_status chp_ctx_destroy(chp_ctx* c) {
  if (!c) return CHP_OK;
  DeviceGuard dg(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->factors) cudaFree(kv.second);
  if (c->scratch) cudaFree(c->scratch);
  if (c->dev_err) cudaFree(c->dev_err);
  chp2d_destroy(c->d2);
  delete c;
  return CHP_OK;
}

// The returned pointer stays valid until the next failing call on the context.
const char* chp_last_error(chp_ctx* c) {
  if (!c) return "null context";
  std::lock_guard<std::mutex> lk(c->mu);
  return c->last_error.c_str();
}

chp_status chp_sysinfo_reset(chp_ctx* c, chp_sys_info* info, int n, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if (!info || n < 0) return fail(c, CHP_ERR_ARG, "bad sysinfo array");
  cudaError_t e = cudaMemsetAsync(info, 0, sizeof(chp_sys_info) * (size_t)n,
                                  (cudaStream_t)stream);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "sysinfo reset");
}

chp_status chp_propagate_hist(chp_ctx* c, const chp_grid* g, const chp_spec* sp, int steps,
                              int nsys, const double* in, long long in_stride, double* out,
                              long long out_stride, const int* sys_index, chp_sys_info* info,
                              double* hist, int hist_len, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why) || !spec_ok(sp, &why)) return fail(c, CHP_ERR_ARG, why);
  if (steps < 1) return fail(c, CHP_ERR_ARG, "steps must be at least 1");
  if (nsys < 0 || !in || !out || !info) return fail(c, CHP_ERR_ARG, "bad arrays");
  if (hist && hist_len < 1) return fail(c, CHP_ERR_ARG, "hist_len must be at least 1");
  if (!hist) hist_len = 0;
  if (sp->scheme != CHP_NONLINEAR_EYRE) { hist = nullptr; hist_len = 0; }
  if (nsys == 0) return CHP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (g->dim == 1) {
    const double* fac = nullptr;
    if (sp->scheme == CHP_LINEAR_B) {
      chp_status s = factor_1d(c, g, sp->dt, sp->b, st, &fac);
      if (s != CHP_OK) return s;
    }
    const size_t per = (size_t)g->m * (size_t)nsys * sizeof(double);
    chp_status s = ensure_scratch(c, per * 9, st);
    if (s != CHP_OK) return s;
    double* ub = c->scratch;
    double* yh = ub + (size_t)g->m * 7 * nsys;
    double* tmp = yh + (size_t)g->m * nsys;
    cudaError_t e = chp1d_propagate(*g, *sp, steps, nsys, in, in_stride, out, out_stride,
                                    sys_index, fac, ub, yh, tmp, info, st, hist, hist_len);
    return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp1d_propagate");
  }
  cudaError_t e = chp2d_propagate(c->d2, *g, *sp, steps, nsys, in, in_stride, out, out_stride,
                                  sys_index, info, hist, hist_len, st, &why);
  if (!why.empty()) return fail(c, CHP_ERR_UNSUPPORTED, why);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp2d_propagate");
}

chp_status chp_propagate(chp_ctx* c, const chp_grid* g, const chp_spec* sp, int steps, int nsys,
                         const double* in, long long in_stride, double* out,
                         long long out_stride, const int* sys_index, chp_sys_info* info,
                         void* stream) {
  return chp_propagate_hist(c, g, sp, steps, nsys, in, in_stride, out, out_stride, sys_index,
                            info, nullptr, 0, stream);
}

chp_status chp_coarse_sweep(chp_ctx* c, const chp_grid* g, const chp_spec* sp, int mode, int nic,
                            int nsl, int n0, int n1, double* U, const double* F, double* G,
                            long long ic_stride, long long sl_stride, unsigned char* changed,
                            double* inc, chp_sys_info* info, void* stream) {
  return chp_coarse_sweep_hop(c, g, sp, mode, nic, nsl, n0, n1, U, F, G, ic_stride, sl_stride,
                              changed, inc, info, nullptr, stream);
}

chp_status chp_coarse_sweep_hop(chp_ctx* c, const chp_grid* g, const chp_spec* sp, int mode, int nic,
                                int nsl, int n0, int n1, double* U, const double* F, double* G,
                                long long ic_stride, long long sl_stride, unsigned char* changed,
                                double* inc, chp_sys_info* info, const chp_hop* hop, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why) || !spec_ok(sp, &why)) return fail(c, CHP_ERR_ARG, why);
  if (mode != 0 && mode != 1) return fail(c, CHP_ERR_ARG, "mode must be 0 or 1");
  if (nic < 1 || nsl < 1 || n0 < 0 || n1 > nsl || n0 > n1)
    return fail(c, CHP_ERR_ARG, "bad slice range");
  if (!U || !G || !info || (mode == 1 && (!F || !changed)))
    return fail(c, CHP_ERR_ARG, "bad arrays");
  if (hop && (!hop->peer_u || !hop->peer_flag || (mode == 1 && !hop->peer_changed)))
    return fail(c, CHP_ERR_ARG, "bad hop descriptor");
  cudaStream_t st = (cudaStream_t)stream;
  const long long fsz = g->dim == 1 ? (long long)g->m : (long long)g->m * g->pitch;
  // the hand-off after (not fused into) the sweep: U[n1] and changed[n1] of every IC
  auto put = [&]() -> chp_status {
    cudaError_t pe = chp_launch_hop_put(fsz, nic, U + (long long)n1 * sl_stride, ic_stride,
                                        mode == 1 ? changed + n1 : nullptr, nsl + 1, *hop, st);
    return pe == cudaSuccess ? CHP_OK : cuda_fail(c, pe, "chp_hop_put");
  };
  if (n0 == n1) return hop ? put() : CHP_OK;
  if (g->dim == 1) {
    const double* fac = nullptr;
    if (sp->scheme == CHP_LINEAR_B) {
      chp_status s = factor_1d(c, g, sp->dt, sp->b, st, &fac);
      if (s != CHP_OK) return s;
    }
    const size_t per = (size_t)g->m * (size_t)nic * sizeof(double);
    chp_status s = ensure_scratch(c, per * 9, st);
    if (s != CHP_OK) return s;
    double* ub = c->scratch;
    double* yh = ub + (size_t)g->m * 7 * nic;
    double* tmp = yh + (size_t)g->m * nic;
    cudaError_t e = chp1d_coarse_sweep(*g, *sp, mode, nic, nsl, n0, n1, U, F, G, ic_stride,
                                       sl_stride, changed, inc, fac, ub, yh, tmp, info, st);
    if (e != cudaSuccess) return cuda_fail(c, e, "chp1d_coarse_sweep");
    return hop ? put() : CHP_OK;
  }
  // the 2D kernels move fields as 16-byte words (rows are N = m + 1 doubles, N even)
  auto odd16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0; };
  if (odd16(U) || odd16(G) || (F && odd16(F)) || (ic_stride & 1) || (sl_stride & 1) ||
      (hop && (odd16(hop->peer_u) || (hop->peer_stride & 1))))
    return fail(c, CHP_ERR_ARG, "2D fields must be 16-byte aligned with even strides");
  bool fused = false;
  cudaError_t e = chp2d_coarse_sweep(c->d2, *g, *sp, mode, nic, nsl, n0, n1, U, F, G, ic_stride,
                                     sl_stride, changed, inc, info, st, &why, hop, &fused);
  if (!why.empty()) return fail(c, CHP_ERR_UNSUPPORTED, why);
  if (e != cudaSuccess) return cuda_fail(c, e, "chp2d_coarse_sweep");
  return (hop && !fused) ? put() : CHP_OK;
}

chp_status chp_hop_wait(chp_ctx* c, const unsigned int* flag, unsigned int seq, void* stream) {
  if (!c || !flag) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  typedef CUresult (*WaitFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<WaitFn>(f);
  }();
  if (!fn) return fail(c, CHP_ERR_UNSUPPORTED, "cuStreamWaitValue32 is not available");
  const CUresult r = fn((CUstream)stream, (CUdeviceptr)(uintptr_t)flag, seq, CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? CHP_OK : fail(c, CHP_ERR_CUDA, "cuStreamWaitValue32 failed");
}

chp_status chp_hop_take(chp_ctx* c, const chp_grid* g, int nic, const double* mail,
                        long long mail_stride, const unsigned char* mail_changed, double* U0,
                        long long ic_stride, unsigned char* changed, long long changed_stride,
                        unsigned int* peer_ack, unsigned int seq, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why)) return fail(c, CHP_ERR_ARG, why);
  if (nic < 1 || !mail || !mail_changed || !U0 || !changed) return fail(c, CHP_ERR_ARG, "bad arrays");
  const long long fsz = g->dim == 1 ? (long long)g->m : (long long)g->m * g->pitch;
  cudaError_t e = chp_launch_hop_take(fsz, nic, mail, mail_stride, mail_changed, U0, ic_stride,
                                      changed, changed_stride, peer_ack, seq, (cudaStream_t)stream);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp_hop_take");
}

chp_status chp_mem_alloc(chp_ctx* c, long long bytes, void** dptr) {
  if (!c || !dptr || bytes <= 0) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  cudaError_t e = cudaMalloc(dptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*dptr, 0, (size_t)bytes);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp_mem_alloc");
}

chp_status chp_mem_free(chp_ctx* c, void* dptr) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  cudaError_t e = cudaFree(dptr);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp_mem_free");
}

chp_status chp_ipc_export(chp_ctx* c, void* dptr, unsigned char* handle64) {
  if (!c || !dptr || !handle64) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "handle size");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dptr);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaIpcGetMemHandle");
  memcpy(handle64, &h, 64);
  return CHP_OK;
}

chp_status chp_ipc_open(chp_ctx* c, const unsigned char* handle64, void** dptr) {
  if (!c || !dptr || !handle64) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "cudaIpcOpenMemHandle");
}

chp_status chp_ipc_close(chp_ctx* c, void* dptr) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  cudaError_t e = cudaIpcCloseMemHandle(dptr);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "cudaIpcCloseMemHandle");
}

chp_status chp_max_abs_diff(chp_ctx* c, const chp_grid* g, int n_fields, const double* a,
                            long long as, const double* b, long long bs, double* out,
                            void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why)) return fail(c, CHP_ERR_ARG, why);
  if (n_fields < 0 || !a || !b || !out) return fail(c, CHP_ERR_ARG, "bad arrays");
  if (n_fields == 0) return CHP_OK;
  cudaError_t e = chp_launch_max_abs_diff(*g, n_fields, a, as, b, bs, out, (cudaStream_t)stream);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "max_abs_diff");
}

chp_status chp_field_stats(chp_ctx* c, const chp_grid* g, int n_fields, const double* in,
                           long long stride, double* out, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why)) return fail(c, CHP_ERR_ARG, why);
  if (n_fields < 0 || !in || !out) return fail(c, CHP_ERR_ARG, "bad arrays");
  if (n_fields == 0) return CHP_OK;
  cudaError_t e = chp_launch_field_stats(*g, n_fields, in, stride, out, (cudaStream_t)stream);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "field_stats");
}

chp_status chp_probe_dfma(chp_ctx* c, int blocks, int iters, double* out, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if (blocks < 1 || iters < 1 || !out) return fail(c, CHP_ERR_ARG, "bad probe arguments");
  cudaError_t e = chp_launch_dfma_probe(blocks, iters, out, (cudaStream_t)stream);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "dfma probe");
}

chp_status chp_nn_propagate(chp_ctx* c, const chp_grid* g, const chp_nn_params* nn, double dt,
                            double eps2, int steps, int nsys, const double* in,
                            long long in_stride, double* out, long long out_stride,
                            const int* sys_index, const double* traces_in, double* traces_out,
                            chp_sys_info* info, void* stream) {
  if (!c) return CHP_ERR_ARG;
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  std::string why;
  if (!grid_ok(g, &why)) return fail(c, CHP_ERR_ARG, why);
  if (!nn) return fail(c, CHP_ERR_ARG, "null nn params");
  // Decomposition / NNParams validation (ddm.py:58-66, 77-93)
  if (g->dim != 1) return fail(c, CHP_ERR_ARG, "domain decomposition is implemented in 1D only");
  if (nn->n_subdomains < 2) return fail(c, CHP_ERR_ARG, "need at least 2 subdomains");
  const int cells = g->nx - 1;
  if (cells % nn->n_subdomains != 0) {
    char buf[160];
    snprintf(buf, sizeof buf, "%d mesh cells do not split evenly into %d subdomains", cells,
             nn->n_subdomains);
    return fail(c, CHP_ERR_ARG, buf);
  }
  if (cells / nn->n_subdomains < 2)
    return fail(c, CHP_ERR_ARG, "subdomains must span at least 2 mesh cells");
  if (!(nn->theta > 0.0 && nn->theta < 1.0))
    return fail(c, CHP_ERR_ARG, "theta must lie in (0, 1)");
  if (!(nn->tol > 0.0) || nn->max_iter < 1)
    return fail(c, CHP_ERR_ARG, "tol must be positive and max_iter at least 1");
  if (nn->n_subdomains > 32)
    return fail(c, CHP_ERR_UNSUPPORTED, "at most 32 subdomains (one warp per system)");
  if (!(dt > 0.0) || !(nn->h2 > 0.0)) return fail(c, CHP_ERR_ARG, "dt and h2 must be positive");
  if (steps < 1) return fail(c, CHP_ERR_ARG, "steps must be at least 1");
  if (nsys < 0 || !in || !out || !info) return fail(c, CHP_ERR_ARG, "bad arrays");
  if (nsys == 0) return CHP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int step = cells / nn->n_subdomains;
  chp_status s = ensure_scratch(c, chp_nn_scratch_bytes(step, nsys, nn->n_subdomains), st);
  if (s != CHP_OK) return s;
  cudaError_t e = chp_nn_launch(*g, *nn, dt, eps2, steps, nsys, in, in_stride, out, out_stride,
                                sys_index, traces_in, traces_out, info, c->scratch, st);
  return e == cudaSuccess ? CHP_OK : cuda_fail(c, e, "chp_nn_propagate");
}

}  // extern "C"

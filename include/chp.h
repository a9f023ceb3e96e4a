/*
 * chp.h -- C ABI of libchp.so, the B200 (sm_100a) implementation of the
 * Parareal / Cahn-Hilliard hot path of arXiv 2304.14074's reference package
 * `chparareal` (/root/reference/pkg/src/chparareal).
 *
 * The reference is pure Python; its plug-in point for this path is the
 * propagator interface `propagate(u, spec, steps, stats)` (schemes.py:321-333)
 * and the four engine call sites that drive it (parareal.py:163, 184, 237,
 * 248).  Every entry point below replaces one of those, batched over systems
 * (initial conditions x time slices).  INTEGRATION.md shows the ctypes
 * binding the Python host layer (paper_2304_14074_b200/_native.py) uses.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (fp64 unless stated); the caller
 *    (PyTorch) owns them.  `stream` is a cudaStream_t passed as void*.
 *  - A 1D field is m contiguous doubles.  A 2D field is m rows of pitch
 *    N = m+1 doubles, x (i) slow, y (j) fast -- the reference's lexicographic
 *    order (grid.py:61-67) -- each row laid out [0, v_1, ..., v_m]: column 0
 *    is the zero Dirichlet boundary, so storage index = math index and rows
 *    are 16-byte aligned.  The pad is ignored on input, written 0 on output.
 *  - Calls are asynchronous on `stream` unless documented otherwise;
 *    per-system outcomes are written to a device `chp_sys_info` array.
 *  - Return codes are chp_status; chp_last_error() gives the message.
 */
#ifndef CHP_H_
#define CHP_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chp_ctx chp_ctx;

typedef enum {
  CHP_OK = 0,
  CHP_ERR_ARG = 1,          /* invalid argument (reference raises ValueError) */
  CHP_ERR_CUDA = 2,         /* CUDA runtime error */
  CHP_ERR_UNSUPPORTED = 3   /* grid/scheme combination not implemented */
} chp_status;

/* Scheme ids -- reference schemes.py:52-58.  NN_LINEAR_A (ddm.py) has its own
 * entry point, chp_nn_propagate, because it carries NN parameters. */
enum { CHP_LINEAR_A = 0, CHP_LINEAR_B = 1, CHP_NONLINEAR_EYRE = 2, CHP_NN_LINEAR_A = 3 };

/* Per-system outcome codes. */
enum {
  CHP_SYS_OK = 0,
  CHP_SYS_NEWTON = 1,     /* NewtonDivergenceError (schemes.py:301-302)      */
  CHP_SYS_NONFINITE = 2,  /* ValueError non-finite field (grid.py:84-85)     */
  CHP_SYS_SINGULAR = 3,   /* zero pivot / not SPD (LinearSolveError)          */
  CHP_SYS_CG = 4,         /* 2D CG budget exhausted (LinearSolveError)        */
  CHP_SYS_NN = 5          /* NNConvergenceError (ddm.py:331-332): fail_iter =
                             sweeps, fail_resid = u-trace increment,
                             newton_maxres = v-trace increment               */
};

/* Spatial grid (grid.py:33-67, operator coefficients of grid.py:98-118). */
typedef struct {
  int dim;        /* 1 or 2 */
  int nx;         /* nodes per axis including the boundary */
  int m;          /* interior points per axis = nx - 2 */
  int pitch;      /* row pitch in doubles (>= m) */
  double h;       /* 1/(nx-1) */
  double hd;      /* h**dim (norm weight, grid.py:149) */
  double c1;      /* Laplacian off-diagonal 1/h^2 (diagonal -2*dim*c1) */
  double s_main;  /* 1D bilaplacian interior diagonal (L@L)[i,i] */
  double s_edge;  /* 1D bilaplacian first/last diagonal */
  double s_off1;  /* 1D bilaplacian first off-diagonal */
  double s_off2;  /* 1D bilaplacian second off-diagonal */
} chp_grid;

/* Propagator spec (schemes.py:61-86); b = eps**2 * dt formed by the caller
 * exactly as the reference forms it (schemes.py:245, 261, 282). */
typedef struct {
  int scheme;
  int newton_max_iter;
  double dt;
  double eps;
  double b;
  double newton_tol;
  double cg_tol;      /* 2D variable-coefficient CG relative tolerance */
  int cg_max_iter;
  int pad_;
} chp_spec;

/* Per-system outcome and Newton aggregates (NewtonStats, schemes.py:100-115). */
typedef struct {
  int status;
  int fail_iter;
  double fail_resid;
  long long newton_steps;
  long long newton_total;
  int newton_max;
  int cg_max;
  double newton_maxres;
  long long cg_total;
} chp_sys_info;

const char* chp_version(void);
const char* chp_status_str(int status);

/* Create a context on `device`: owns cached solver tables (the analogue of
 * schemes._FACTOR_CACHE, schemes.py:134-142) and scratch.  One per device per
 * process.  Every entry point locks the context (calls from several host
 * threads serialise; the reference calls propagate from worker threads,
 * SPEC.md:163) and runs on the context's device whatever device is current,
 * restoring the caller's current device on return; `stream` must belong to that
 * device. */
chp_status chp_ctx_create(int device, chp_ctx** out);
chp_status chp_ctx_destroy(chp_ctx* ctx);
const char* chp_last_error(chp_ctx* ctx);

/* Zero every chp_sys_info of an array (async). */
chp_status chp_sysinfo_reset(chp_ctx* ctx, chp_sys_info* info, int n, void* stream);

/*
 * chp_propagate -- `steps` steps of spec->scheme on `nsys` fields.
 * Replaces schemes.propagate (schemes.py:321-333) and the step functions
 * step_linear_a / step_linear_b / step_nonlinear (schemes.py:235-305).
 * System s reads in + idx(s)*in_stride and writes out + idx(s)*out_stride,
 * idx(s) = sys_index ? sys_index[s] : s  (sys_index: device int array).
 * in == out is allowed.  info[idx(s)] accumulates the outcome.
 */
chp_status chp_propagate(chp_ctx* ctx, const chp_grid* g, const chp_spec* spec,
                         int steps, int nsys,
                         const double* in, long long in_stride,
                         double* out, long long out_stride,
                         const int* sys_index, chp_sys_info* info, void* stream);

/*
 * chp_coarse_sweep -- the sequential coarse recursion of parareal.py:245-251
 * (mode 1) or the coarse initialisation of parareal.py:182-185 (mode 0), for
 * `nic` independent initial conditions over slices [n_begin, n_end).
 *
 * Layout (per IC i, slice n): U  + i*ic_stride + n*slice_stride  (N+1 slots)
 *                             F  + i*ic_stride + n*slice_stride  (N slots)
 *                             G  + i*ic_stride + n*slice_stride  (N slots)
 * mode 0: U[n+1] = G(U[n]);  G[n] = U[n+1]                   (coarse_init)
 * mode 1: g = G(U[n]) (reused from G[n] when U[n] is bit-identical to its
 *         previous value, i.e. changed[n]==0);
 *         U[n+1] = (g + F[n]) - G[n];  G[n] = g             (parareal.py:249)
 *         changed[n+1] = any bit of U[n+1] differs; inc[i] = max |dU|.
 * `changed` (device uint8, nic*(N+1)) must hold changed[i*(N+1)+n_begin] on
 * entry (1 iff U[n_begin] changed during this sweep).  Bit 1 of
 * changed[i*(N+1)] (slot 0 -- U[0] never changes) freezes IC i: it is skipped.
 * `inc` (device double, nic) is max-accumulated.
 * 2D grids: the kernels move fields as 16-byte words, so U, F, G (and a hop mailbox)
 * must be 16-byte aligned and both strides even (CHP_ERR_ARG otherwise).
 */
chp_status chp_coarse_sweep(chp_ctx* ctx, const chp_grid* g, const chp_spec* coarse,
                            int mode, int nic, int nslices, int n_begin, int n_end,
                            double* U, const double* F, double* G,
                            long long ic_stride, long long slice_stride,
                            unsigned char* changed, double* inc,
                            chp_sys_info* info, void* stream);

/*
 * Device-initiated boundary hand-off of the sharded coarse chain (SURVEY.md 8(e),
 * 8(f2); replaces the per-hop dist.send/recv of the slice end state around the
 * sequential sweep of parareal.py:245-251).  The sending rank's sweep stores
 * U[n_end] of every IC, and its "changed in this sweep" flags, straight into a
 * mailbox in the receiving rank's memory (a peer mapping: cudaIpc between
 * processes, or plain device memory for shards on one device) and then releases
 * *peer_flag = seq (system scope).  In the 2D LINEAR_A cooperative kernel the stores
 * are fused into the last slice's correction; other coarse paths run a put kernel
 * after the sweep.  The receiver's stream waits on its flag (chp_hop_wait: a
 * stream memory operation, no kernel spins), takes the mailbox (chp_hop_take) and
 * acknowledges by releasing `seq` into the sender's ack word.
 */
typedef struct {
  double* peer_u;               /* IC i's field goes to peer_u + i * peer_stride */
  long long peer_stride;
  unsigned char* peer_changed;  /* nic bytes: bit 0 of changed[i][n_end] */
  unsigned int* peer_flag;      /* released with seq after the data */
  unsigned int seq;
  unsigned int pad_;
} chp_hop;

/* chp_coarse_sweep followed by (or fused with) the hand-off described by `hop`
 * (hop == NULL: exactly chp_coarse_sweep). */
chp_status chp_coarse_sweep_hop(chp_ctx* ctx, const chp_grid* g, const chp_spec* coarse,
                                int mode, int nic, int nslices, int n_begin, int n_end,
                                double* U, const double* F, double* G,
                                long long ic_stride, long long slice_stride,
                                unsigned char* changed, double* inc,
                                chp_sys_info* info, const chp_hop* hop, void* stream);

/* Work queued on `stream` after this call starts once *flag >= seq (flag: device
 * memory of this context's device; cuStreamWaitValue32, no kernel). */
chp_status chp_hop_wait(chp_ctx* ctx, const unsigned int* flag, unsigned int seq, void* stream);

/* Take a received boundary: for every IC whose freeze bit (bit 1 of changed[i *
 * changed_stride]) is clear, U0[i * ic_stride] = mail[i * mail_stride] and bit 0 of
 * changed[i * changed_stride] = bit 0 of mail_changed[i]; then release *peer_ack =
 * seq (peer_ack may be NULL). */
chp_status chp_hop_take(chp_ctx* ctx, const chp_grid* g, int nic, const double* mail,
                        long long mail_stride, const unsigned char* mail_changed, double* U0,
                        long long ic_stride, unsigned char* changed, long long changed_stride,
                        unsigned int* peer_ack, unsigned int seq, void* stream);

/* Mailbox memory: plain cudaMalloc allocations (zero-filled) that can be shared with
 * another process on the node.  handle: 64 bytes (cudaIpcMemHandle_t). */
chp_status chp_mem_alloc(chp_ctx* ctx, long long bytes, void** dptr);
chp_status chp_mem_free(chp_ctx* ctx, void* dptr);
chp_status chp_ipc_export(chp_ctx* ctx, void* dptr, unsigned char* handle64);
chp_status chp_ipc_open(chp_ctx* ctx, const unsigned char* handle64, void** dptr);
chp_status chp_ipc_close(chp_ctx* ctx, void* dptr);

/* max |a - b| over n_fields fields of `size` entries (row pitch aware),
 * max-accumulated into out[0] (device). */
chp_status chp_max_abs_diff(chp_ctx* ctx, const chp_grid* g, int n_fields,
                            const double* a, long long a_stride,
                            const double* b, long long b_stride,
                            double* out, void* stream);

/*
 * chp_field_stats -- the sums behind l2_norm, energy and mass (grid.py:147-181)
 * for n_fields fields (field f at in + f*stride), one fixed-order device
 * reduction per field (bitwise reproducible).  out (device, 4*n_fields doubles):
 * out[4f] = sum v^2, out[4f+1] = sum (v^2-1)^2, out[4f+2] = sum of squared
 * differences along every axis with the Dirichlet zeros at both ends
 * (grid.py:168-175), out[4f+3] = sum v.
 */
chp_status chp_field_stats(chp_ctx* ctx, const chp_grid* g, int n_fields, const double* in,
                           long long stride, double* out, void* stream);

/*
 * chp_propagate_hist -- chp_propagate that also records StepReport.residual_history
 * (schemes.py:285-290) of a NONLINEAR_EYRE propagation: for every system idx(s),
 * hist[idx * hist_len + it] = the residual norm before Newton solve `it`
 * (it < hist_len) of its last step; entries after the accepted (or failing)
 * iteration are left untouched.  `hist` (caller-owned device buffer, or NULL) is
 * used by this call only; other schemes ignore it.  Replaces the per-step
 * report of step_nonlinear (schemes.py:270-305).
 */
chp_status chp_propagate_hist(chp_ctx* ctx, const chp_grid* g, const chp_spec* spec,
                              int steps, int nsys,
                              const double* in, long long in_stride,
                              double* out, long long out_stride,
                              const int* sys_index, chp_sys_info* info,
                              double* hist, int hist_len, void* stream);

/* Neumann-Neumann interface-iteration parameters (ddm.py:51-66, NNParams)
 * plus h**2 formed by the caller as grid.h**2 (ddm.py:274). */
typedef struct {
  int n_subdomains;   /* >= 2, divides nx - 1, (nx-1)/n >= 2; <= 32 here */
  int max_iter;       /* sweep budget */
  int warm_start;     /* carry the traces from step to step (ddm.py:367-371) */
  int pad_;
  double theta;       /* relaxation in (0, 1) */
  double tol;         /* stop when both trace increments <= tol */
  double h2;          /* grid.h**2 */
} chp_nn_params;

/*
 * chp_nn_propagate -- `steps` Neumann-Neumann steps (Scheme.NN_LINEAR_A) on
 * `nsys` 1D fields.  Replaces ddm.nn_propagate (ddm.py:360-372), hence
 * schemes.propagate's NN_LINEAR_A branch (schemes.py:326-329); with steps = 1
 * and traces it is ddm._nn_solve (ddm.py:268-340).  eps2 = eps**2 formed by
 * the caller (ddm.py:275).  Fields/strides/sys_index/info as chp_propagate.
 * traces_in (optional, device, nsys' x 2 x (n-1) doubles indexed by idx(s):
 * g then h) seeds the first step's traces (zeros when NULL); traces_out
 * (optional) receives the final step's converged traces.  info: newton_steps
 * += steps, newton_total += interface sweeps, newton_max = max sweeps per
 * step, newton_maxres = max accepted trace increment.
 */
chp_status chp_nn_propagate(chp_ctx* ctx, const chp_grid* g, const chp_nn_params* nn,
                            double dt, double eps2, int steps, int nsys,
                            const double* in, long long in_stride,
                            double* out, long long out_stride, const int* sys_index,
                            const double* traces_in, double* traces_out,
                            chp_sys_info* info, void* stream);

/* Measurement: `blocks` x 256 threads each running 16 independent DFMA chains of
 * `iters` steps (2*16*iters flop per thread) -- the FP64 peak the 1D configs' flop
 * model is reported against (bench.py).  `out`: one device double (scratch). */
chp_status chp_probe_dfma(chp_ctx* ctx, int blocks, int iters, double* out, void* stream);

/* Debug: barrier timestamps (globaltimer ns) of the last cooperative 2D
 * coarse sweep when CHP_COOP_TRACE is set in the environment; returns the
 * number of entries copied (0 when tracing is off). */
int chp_debug_trace(unsigned long long* host, int n);

#ifdef __cplusplus
}
#endif
#endif /* CHP_H_ */

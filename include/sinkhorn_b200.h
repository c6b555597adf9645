/*
 * sinkhorn_b200.h -- C ABI of the B200-native batched log-domain Sinkhorn loss.
 *
 * Drop-in boundary for the reference's FFI (`/root/reference/pkg/frontend/src/ffi.ts`).
 * Plain C types only: no torch, no C++ in the signatures.  The library is
 * `paper_1907_01729_b200/_lib/libsinkhorn_b200.so` (built by __graft_entry__.build()).
 *
 * Two layers:
 *
 *  1. Host-buffer entry points with the reference's exact semantics
 *     (row-major float64 views, outputs written in place, integer status,
 *     nothing thrown).  `sinkhorn_forward_v1` replaces ffi.ts:80-134 and
 *     `sinkhorn_backward_v1` replaces ffi.ts:143-191.  They copy the views to
 *     the GPU, run the fp32 device pipeline below and copy results back.
 *
 *  2. Device entry points (`*_device_v1`) over float32 device pointers,
 *     stream-ordered on a caller-supplied cudaStream_t, with caller-owned
 *     workspace.  These are what the PyTorch layer binds (ctypes) and what
 *     extends the reference: per-sample costs, on-the-fly grid costs,
 *     iteration count / residual outputs, partial (max, sum-exp) outputs for
 *     row-sharded multi-GPU solves, and the transport-plan gradient dC.
 *
 * Status codes: ffi.ts:21-25 (0, 10-13) plus extensions 14-21 (the reference
 * raises exceptions for these).
 */
#ifndef SINKHORN_B200_H
#define SINKHORN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SINKHORN_STATUS_OK 0                /* ffi.ts:21 STATUS_OK */
#define SINKHORN_STATUS_SHAPE_MISMATCH 10   /* ffi.ts:22 */
#define SINKHORN_STATUS_INVALID_HISTOGRAM 11/* ffi.ts:23 (core.py:143-160 rules) */
#define SINKHORN_STATUS_NON_FINITE_OUTPUT 12/* ffi.ts:24; also NaN state (batch.py:326-327) */
#define SINKHORN_STATUS_ZERO_MASS_LANE 13   /* ffi.ts:25; batch.py:366-370 */
#define SINKHORN_STATUS_INVALID_CONFIG 14   /* core.py:88-96 ValueError */
#define SINKHORN_STATUS_INVALID_COST 15     /* core.py:53-63 ValueError */
#define SINKHORN_STATUS_BAD_ARGUMENT 16     /* null pointer / unsupported descriptor */
#define SINKHORN_STATUS_WORKSPACE 17        /* workspace too small */
#define SINKHORN_STATUS_EXACT_NEEDED 18     /* row-sharded GEMM solve: rerun exactly (see below) */
#define SINKHORN_STATUS_CUDA_ERROR 20       /* CUDA runtime error (message: sinkhorn_last_error) */

/* ---- layer 1: host float64 views (ffi.ts:14-19 TensorView) ------------- */

/* Row-major contiguous view. `length` is the number of elements available at
 * `data` (ffi.ts:33-38 checks offset + size <= data.length; fold any offset
 * into `data`). */
typedef struct sinkhorn_view_v1 {
  double* data;
  int32_t ndim;
  int64_t shape[2];
  int64_t length;
} sinkhorn_view_v1;

/* Replaces ffi.ts:80-134 sinkhorn_forward_v1.  Shapes: mu (B,d1), nu (B,d2),
 * cost (d1,d2), out_cost (B,), out_log_u (B,d1), out_log_v (B,d2).
 * check_interval is 10, the CLI default the reference's runner inherits
 * (runner.ts:48-55, cli.py:50).  B == 0 is a successful no-op. */
int32_t sinkhorn_forward_v1(const sinkhorn_view_v1* mu, const sinkhorn_view_v1* nu,
                            const sinkhorn_view_v1* cost, double lambda, int32_t max_iters,
                            double tolerance, const sinkhorn_view_v1* out_cost,
                            const sinkhorn_view_v1* out_log_u, const sinkhorn_view_v1* out_log_v);

/* Replaces ffi.ts:143-191 sinkhorn_backward_v1.  Shapes: log_u (B,d1),
 * log_v (B,d2), upstream (B,), out_grad_mu (B,d1), out_grad_nu (B,d2).
 * Any -inf potential returns 13 (ffi.ts:177-179). */
int32_t sinkhorn_backward_v1(const sinkhorn_view_v1* log_u, const sinkhorn_view_v1* log_v,
                             double lambda, const sinkhorn_view_v1* upstream,
                             const sinkhorn_view_v1* out_grad_mu,
                             const sinkhorn_view_v1* out_grad_nu);

/* ---- layer 2: device float32 pipeline ----------------------------------- */

#define SINKHORN_COST_SHARED 0     /* one stored (d1,d2) cost for all lanes (the reference's case) */
#define SINKHORN_COST_PER_SAMPLE 1 /* stored (B,d1,d2), one cost per lane (BASELINE config 4) */
#define SINKHORN_COST_POINTS 3     /* squared Euclidean between point clouds x (d1, D), y (d2, D):
                                      cost points to [x; y], (d1 + d2) x D fp32, D in grid_nx;
                                      |x|^2 + |y|^2 - 2 x.y with the x.y contraction on the
                                      tensor cores */
#define SINKHORN_COST_GRID2D 2     /* squared Euclidean on an nx*ny grid, never materialised
                                      (BASELINE config 3); d1 = d2 = nx*ny,
                                      point k at ((k % nx)*hx, (k / nx)*hy) */

typedef struct sinkhorn_problem_v1 {
  int64_t B, d1, d2;
  int32_t cost_kind;     /* SINKHORN_COST_* */
  int32_t grid_nx, grid_ny;
  float grid_hx, grid_hy;
} sinkhorn_problem_v1;

#define SINKHORN_FLAG_SKIP_VALIDATION 1u /* trust mu/nu/cost (caller validated) */
#define SINKHORN_FLAG_PARTIAL_ROWS 2u    /* reserved: row-sharded solves use the half-sweep API */
#define SINKHORN_FLAG_TIME_LOOP 4u       /* record CUDA events around the iteration loop */
#define SINKHORN_FLAG_EXACT_MAX 8u       /* always two-pass chunks (no previous-lse estimate) */
#define SINKHORN_FLAG_MUFU_ONLY 16u      /* every exponential on MUFU (no FMA-pipe polynomial) */
#define SINKHORN_FLAG_PERSISTENT 32u     /* shared/grid costs: whole loop in one cooperative kernel */
#define SINKHORN_FLAG_TILED_ONLY 64u     /* never take the single-launch small-problem solver */
#define SINKHORN_FLAG_DENSE_GRID 128u    /* grid costs: dense on-the-fly sweeps, not separable */
#define SINKHORN_FLAG_NO_FUSED 256u      /* shared costs: two half-sweeps per iteration, not the
                                            fused row->column pass (sweep_fused.cuh) */
#define SINKHORN_FLAG_NO_GEMM 512u       /* large shared costs: tiled half-sweeps, not the two
                                            fp32 GEMMs per iteration (sweep_gemm.cuh) */
#define SINKHORN_FLAG_FORCE_GEMM 1024u   /* shared costs: the GEMM path even where the fused
                                            pass applies (d <= 1024) */
#define SINKHORN_FLAG_TIME_KERNEL 2048u  /* CUDA events around each launch of the solve's
                                            dominant kernel (sinkhorn_last_kernel_ms_v1) */
#define SINKHORN_FLAG_FORCE_RERUN 4096u  /* diagnostics: behave as if an estimate guard fired
                                            (exercises the exact rerun, sync and async) */

typedef struct sinkhorn_options_v1 {
  double lambda;          /* > 0, finite */
  int32_t max_iters;      /* >= 1 */
  int32_t check_interval; /* >= 1 (reference default 10) */
  double tolerance;       /* >= 0; 0 runs exactly max_iters iterations */
  uint32_t flags;
} sinkhorn_options_v1;

/* Bytes of device workspace sinkhorn_forward_device_v1 needs for `prob`. */
size_t sinkhorn_workspace_bytes_v1(const sinkhorn_problem_v1* prob);

/* batch_forward (batch.py:264-349) on the GPU.  All pointers are device
 * pointers; mu (B,d1), nu (B,d2) row-major; cost (d1,d2) for SHARED,
 * (B,d1,d2) for PER_SAMPLE, ignored for GRID2D.  Outputs: out_cost (B,),
 * out_log_u (B,d1), out_log_v (B,d2) natural-log potentials; optional
 * out_iterations (1 int32, host or device memory: host) and out_residuals (B,)
 * may be NULL.  `stream` is a cudaStream_t (NULL = legacy default stream).
 * Synchronises `stream` once at the end (and at every convergence check when
 * tolerance > 0) to report the status. */
int32_t sinkhorn_forward_device_v1(const sinkhorn_problem_v1* prob,
                                   const sinkhorn_options_v1* opt, const float* mu,
                                   const float* nu, const float* cost, float* out_cost,
                                   float* out_log_u, float* out_log_v, int32_t* out_iterations,
                                   float* out_residuals, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* float64 parity mode: the reference's float64 iteration
 * (batch.py:264-349) on the device, in natural log, reaching the
 * reference's default tolerance 1e-9 (core.py:85) that an fp32 solve cannot.
 * Same problem / options / statuses as sinkhorn_forward_device_v1, with
 * double device buffers and its own workspace size.  Slower than the fp32
 * paths: one warp per output, exact two-pass log-sum-exp in double. */
size_t sinkhorn_workspace_bytes_f64_v1(const sinkhorn_problem_v1* prob);
int32_t sinkhorn_forward_f64_device_v1(const sinkhorn_problem_v1* prob,
                                       const sinkhorn_options_v1* opt, const double* mu,
                                       const double* nu, const double* cost, double* out_cost,
                                       double* out_log_u, double* out_log_v,
                                       int32_t* out_iterations, double* out_residuals,
                                       void* workspace, size_t workspace_bytes, void* stream);
/* batch_backward in float64 over device buffers (the fp64 mode's backward). */
int32_t sinkhorn_backward_f64_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                        const double* log_u, const double* log_v,
                                        const double* upstream, double* out_grad_mu,
                                        double* out_grad_nu, int32_t* out_zero_mass_lane,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* Warm start (the reference has no such API, batch.py:295
 * always starts from log_u = 0 on the support): as sinkhorn_forward_device_v1,
 * but the iteration starts from init_log_u (B, d1) natural log, device fp32,
 * kept -inf off the support.  init_log_u == NULL is a cold start.  Running
 * k1 iterations, then k2 more from the returned log_u, equals one run of
 * k1 + k2 iterations. */
int32_t sinkhorn_forward_warm_device_v1(const sinkhorn_problem_v1* prob,
                                        const sinkhorn_options_v1* opt, const float* mu,
                                        const float* nu, const float* cost,
                                        const float* init_log_u, float* out_cost,
                                        float* out_log_u, float* out_log_v,
                                        int32_t* out_iterations, float* out_residuals,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* batch_backward (batch.py:352-375): grad = upstream[b]*lambda*(x - mean_i x).
 * Any -inf in a lane returns 13; `out_zero_mass_lane` (host, may be NULL)
 * receives the first such lane.  No workspace beyond 64 bytes (passed). */
int32_t sinkhorn_backward_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                    const float* log_u, const float* log_v,
                                    const float* upstream, float* out_grad_mu,
                                    float* out_grad_nu, int32_t* out_zero_mass_lane,
                                    void* workspace, size_t workspace_bytes, void* stream);

/* One half-sweep, fused_log_reduction (batch.py:208-230):
 * out[b,j] = target[b,j] - logsumexp_i(-cost[i,j]/lambda + log_x[b,i]),
 * shapes log_x (B,d1), cost (d1,d2), target (B,d2), out (B,d2), natural log.
 * With out_max/out_sum non-NULL the (max, sum) accumulator pairs of the
 * reduction are emitted instead (log base 2: lse = max + log2(sum)), which is
 * the partial state a row-sharded solve merges across GPUs
 * (OnlineLseAccumulator.merge, batch.py:116-130); `out` may then be NULL.
 * Workspace: sinkhorn_half_sweep_workspace_bytes_v1. */
size_t sinkhorn_half_sweep_workspace_bytes_v1(int64_t B, int64_t d1, int64_t d2);
int32_t sinkhorn_half_sweep_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                      const float* log_x, const float* cost,
                                      const float* target, float* out, float* out_max,
                                      float* out_sum, void* workspace, size_t workspace_bytes,
                                      void* stream);

/* Per-lane log2 of sum_{i,j} P[i,j] * c[i,j] over the given cost rows: the
 * E0 partial a row-sharded solve merges across GPUs by log-sum-exp
 * (batch.py:331-337 restricted to a row block).  Natural-log inputs
 * log_u (B,d1), log_v (B,d2); out_log2 (B,).  Workspace as the half-sweep. */
int32_t sinkhorn_e0_partial_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                      const float* log_u, const float* log_v, const float* cost,
                                      float* out_log2, void* workspace, size_t workspace_bytes,
                                      void* stream);

/* Cross-process agreement on the stopping test (batch-sharded lockstep,
 * batch.py:318-322): when set (per thread), every convergence check calls
 * fn(local max residual, user) and stops iff the returned global max <= tol.
 * All ranks call it the same number of times: once per check, plus once at
 * the end of a solve's first attempt with local_max = 1 if this rank's
 * estimate-mode sweeps need the exact rerun (else 0), so that the ranks rerun
 * together or not at all.  NULL restores local checks. */
typedef double (*sinkhorn_residual_reducer_v1)(double local_max, void* user);
void sinkhorn_set_residual_reducer_v1(sinkhorn_residual_reducer_v1 fn, void* user);

/* Asynchronous forward (tolerance 0 only; SPEC.md:515-516 reentrancy, no host
 * synchronisation -- SURVEY 8(b) "none with tol=0").  Same arguments as
 * sinkhorn_forward_device_v1 minus out_iterations (= max_iters), plus a device
 * int32 the library writes the final status to, in stream order: the call
 * returns once the solve is enqueued.  Host-detectable errors (shapes,
 * config, null pointers, workspace) are still returned.  Device-detected
 * statuses (11 histogram, 12 non-finite, 15 cost) land in *device_status.  The
 * estimate-guard rerun is decided on the device: a conditional graph node runs
 * the exact solve (captured once per pointers/problem and replayed) only when
 * a guard fired.  Workspace and outputs must stay alive until the stream
 * reaches the solve's end. */
int32_t sinkhorn_forward_async_device_v1(const sinkhorn_problem_v1* prob,
                                         const sinkhorn_options_v1* opt, const float* mu,
                                         const float* nu, const float* cost, float* out_cost,
                                         float* out_log_u, float* out_log_v,
                                         float* out_residuals, int32_t* device_status,
                                         void* workspace, size_t workspace_bytes, void* stream);

/* Row-sharded solves (BASELINE config 5 across GPUs).  Rank r
 * owns rows I_r of the shared cost and of mu / log u; every rank holds the
 * full nu and log v.  The library runs the GEMM iteration (sweep_gemm.cuh,
 * contractions on the tensor cores) on the rank's rows and calls `allreduce`
 * -- enqueue-only, on `stream`, no host synchronisation -- once per column
 * sweep to sum the ranks' column partials (B*d2 floats), and once for the
 * per-lane E0 partials (B floats).  With a common per-lane shift (every rank
 * holds log v) the (max, sum-exp) merge of batch.py:116-130 reduces to that
 * one sum.  Convergence checks (tolerance > 0) and the estimate-guard
 * decision go through the residual reducer (sinkhorn_set_residual_reducer_v1),
 * which the caller sets to a MAX over ranks.  prob->d1 is the rank's row
 * count; mu_rows (B, d1), cost_rows (d1, d2); out_log_u_rows (B, d1).  The
 * caller validates the histograms globally (a slice of mu does not sum to 1).
 * Status 18 (SINKHORN_STATUS_EXACT_NEEDED, on every rank together): a range
 * guard fired (sums below 2^-60); rerun the solve with the exact log-domain
 * half-sweeps (sinkhorn_half_sweep_device_v1). */
#define SINKHORN_REDUCE_SUM 0
typedef void (*sinkhorn_allreduce_v1)(float* data, int64_t count, int32_t op, void* stream,
                                      void* user);
int32_t sinkhorn_forward_rows_device_v1(const sinkhorn_problem_v1* prob,
                                        const sinkhorn_options_v1* opt, const float* mu_rows,
                                        const float* nu, const float* cost_rows,
                                        float* out_cost, float* out_log_u_rows, float* out_log_v,
                                        int32_t* out_iterations, float* out_residuals,
                                        sinkhorn_allreduce_v1 allreduce, void* user,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* Transport-plan gradient w.r.t. the cost (north-star item 4, core.py:363-368):
 * SHARED:     dC[i,j]   = sum_b upstream[b] * P_b[i,j]
 * PER_SAMPLE: dC[b,i,j] = upstream[b] * P_b[i,j]
 * with P_b[i,j] = exp(log_u[b,i] - c[i,j]/lambda + log_v[b,j]): the envelope
 * gradient dE^lambda/dC = P, the same multiplier convention as the histogram
 * gradient (pkg/docs/KNOWN-FAILURES.md:14-22); see DESIGN.md.
 * GRID2D is rejected (no materialised cost to differentiate). */
int32_t sinkhorn_plan_grad_device_v1(const sinkhorn_problem_v1* prob, double lambda,
                                     const float* log_u, const float* log_v, const float* cost,
                                     const float* upstream, float* out_grad_cost, void* stream);

/* The same dC with a caller workspace: shared costs run it as a tensor-core
 * contraction over the lanes, S = U^T V with U_bi = up_b 2^(log2 u_bi - max_b),
 * V_bj = 2^(log2 v_bj - max_b) (3xTF32 on tcgen05), then dC_ij = S_ij *
 * 2^(-c_ij/lambda log2e + the two shifts).  Other cost kinds fall back to
 * sinkhorn_plan_grad_device_v1. */
size_t sinkhorn_plan_grad_workspace_bytes_v1(const sinkhorn_problem_v1* prob);
int32_t sinkhorn_plan_grad_ws_device_v1(const sinkhorn_problem_v1* prob, double lambda,
                                        const float* log_u, const float* log_v, const float* cost,
                                        const float* upstream, float* out_grad_cost,
                                        void* workspace, size_t workspace_bytes, void* stream);

/* Human-readable detail for the last non-zero status on this thread. */
const char* sinkhorn_last_error(void);

/* Library version string ("paper_1907_01729_b200 <semver> sm_100a"). */
const char* sinkhorn_version(void);

/* Instrumentation (benchmarks): kernels launched by this thread so far, and
 * the elapsed milliseconds (CUDA events on the caller's stream) of the last
 * iteration loop run with SINKHORN_FLAG_TIME_LOOP (-1 if none). */
unsigned long long sinkhorn_launch_count_v1(void);
/* Solves this thread redid in exact two-pass mode because a previous-lse
 * estimate overshot the result (estimate mode). */
unsigned long long sinkhorn_exact_reruns_v1(void);
float sinkhorn_last_loop_ms_v1(void);
/* Total milliseconds (CUDA events) and launch count of the dominant kernel's
 * launches in this thread's last forward run with SINKHORN_FLAG_TIME_KERNEL:
 * umma_gemm_kernel (GEMM path), fused_ps_kernel / fgemm_pass_kernel /
 * fused_pass_kernel (fused passes), tiled_sweep_kernel, sep_sweep_kernel,
 * small_solve_kernel.  -1 ms if none. */
float sinkhorn_last_kernel_ms_v1(int32_t* launches);
/* Solver path of this thread's last forward: "small" (one-launch solve,
 * cost in shared memory), "tiled" (stream-K sweeps), "persistent" (opt-in
 * cooperative loop) or "lane" (per-sample costs). */
const char* sinkhorn_last_path_v1(void);   /* ... or "separable" (grid costs) */

#ifdef __cplusplus
}
#endif

#endif /* SINKHORN_B200_H */

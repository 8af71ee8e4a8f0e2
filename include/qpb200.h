/*
 * qpb200.h — C ABI of the B200 (sm_100a) batched f32 interior-point QP solver
 * with implicit (spectrally bounded) complementarity, arxiv 2605.17913.
 *
 * Citations: "P:L" = PAPER.md line L (section / equation / algorithm given),
 * "S:L" = SPEC.md line L, "Qn" = a reading of the paper listed in DESIGN.md §2.
 *
 * The library solves, for every problem b of a batch, the QP of Eq. 1-2
 *
 *      minimize ½ xᵀQx + qᵀx   s.t.  A x = b,  G x ≤ h   (x ∈ ℝⁿ, A: m×n, G: p×n)
 * with Algorithm 1, and differentiates the solution with
 * Algorithm 2 (relaxation to κ_relax) followed by Algorithm 3
 * (implicit-function-theorem gradients; sign reading Q7).
 *
 * Memory and layout (all entry points):
 *   - f32, batch-major, row-major, contiguous: Q[B][n][n], q[B][n], A[B][m][n],
 *     b[B][m], G[B][p][n], h[B][p].  The batch stride of each data tensor is
 *     given in qp_dims (in elements); a stride of 0 marks a tensor SHARED by
 *     all problems of the batch (end-to-end learning, BASELINE config 4).
 *   - Q must be symmetric (Q ∈ 𝕊ⁿ₊).  It is not symmetrised.
 *   - Pointers must be 4-byte aligned (QP_ERR_ALIGN otherwise).
 *   - qp_config.mem_kind == QP_MEM_DEVICE: every pointer is device memory of
 *     the ctx's device; calls are asynchronous and stream-ordered on the ctx
 *     stream; the caller synchronises.  QP_MEM_HOST: every pointer is host
 *     memory (ideally pinned); the library copies in and out through its own
 *     device staging buffers and the call returns after the results are back
 *     in host memory.  QP_MEM_HOST_ASYNC: as QP_MEM_HOST, but the calls only
 *     enqueue their copies and kernels on the ctx stream (and, on path 1, its
 *     eight chunk streams, joined back into the ctx stream); host outputs are
 *     valid, and host inputs may be modified, once the ctx stream has been
 *     synchronised.  A backward call may then start on the problems whose
 *     solve chunk has finished while later chunks still run.
 *   - All buffers are caller-owned.  The ctx owns its workspaces only.
 *   - qp_backward_batched reuses the problem data and the solution of the
 *     LAST qp_solve_batched call on the same ctx: with QP_MEM_DEVICE the
 *     caller must keep Q…h and x, s, z, y alive and unmodified in between
 *     (autograd saved-tensor semantics); with QP_MEM_HOST the ctx keeps device
 *     copies itself.
 *
 *   - Path 4 (qp_info.path, the batched engine for large shapes) reads back,
 *     after each Newton iteration, how many problems still iterate: its calls
 *     return when the work is complete (the ctx stream is synchronised), still
 *     stream-ordered after earlier work on that stream.
 *
 * Errors: an API-level qp_err return covers argument, shape and CUDA errors.
 * The numerical outcome is per problem in status[] and never aborts a call
 * (S:262): a failed problem keeps its last finite iterate, its gradients are
 * zero-filled and its status says why.
 */
#ifndef QPB200_H
#define QPB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QP_OK = 0,
  QP_ERR_INVALID_ARG = -1,  /* null pointer where required, bad config value   */
  QP_ERR_SHAPE = -2,        /* n < 1, negative m/p, or n+p+m beyond the kernels */
  QP_ERR_ALIGN = -3,        /* pointer not 4-byte aligned                        */
  QP_ERR_CUDA = -4,         /* a CUDA runtime call failed                        */
  QP_ERR_OOM = -5,          /* workspace allocation failed                       */
  QP_ERR_NOT_SOLVED = -6,   /* backward before any solve on this ctx             */
  QP_ERR_UNSUPPORTED = -7   /* option not available for this size / formulation */
} qp_err;

/* Per-problem status (low byte; numbers mirror S:484) and failure stage
 * (bits 8..15; the Table 1 categories of P:1009-1013). */
enum { QP_CONVERGED = 0, QP_MAX_ITER = 2, QP_NUMERICAL_FAILURE = 3 };
enum {
  QP_STAGE_NONE = 0, QP_STAGE_SCALING = 1, QP_STAGE_PREDICTOR = 2, QP_STAGE_CENTERING = 3,
  QP_STAGE_CORRECTOR = 4, QP_STAGE_LINESEARCH = 5, QP_STAGE_RELAX = 6, QP_STAGE_BACKWARD = 7,
  QP_STAGE_INIT = 8
};

enum { QP_IMPLICIT = 0, QP_EXPLICIT = 1 };   /* formulation: Eq. 14 or Eq. 8 */
enum { QP_MEM_DEVICE = 0, QP_MEM_HOST = 1, QP_MEM_HOST_ASYNC = 2 };
/* Alg. 2's linear solves (qp_config.relax_mode): exact Newton, a fresh
 * factorisation per step (reading Q6); or the guarded chord of SURVEY §8(f)
 * N2(i) (reading Q26): the solve caches the factorisation of its first
 * iterate with κ < √10·κ_relax ("the matrix factorizations K̃ computed during
 * the forward solve ... can be heavily reused"; "if K̃ not cached",
 * P:513) and Alg. 2 takes chord steps on it — the current residuals, the
 * cached Jacobian — while each shrinks ψ = max(φ, |κ/κ_relax − 1|) by
 * chord_rho (at most chord_max of them); from the first that does not it
 * takes exact Newton steps.  A chord phase ends only at φ ≤ relax_tol.
 * Either way the final factorisation is at the relaxed point, so Alg. 3's
 * gradients are the exact IFT gradients there.  Paths 1 and 4 (paths 2/3
 * and the standard arm relax by exact Newton; so does a batch whose cache —
 * one factor per problem — would not fit in a quarter of the free device
 * memory); qp_info.relax_mode reports the mode in effect. */
enum { QP_RELAX_NEWTON = 0, QP_RELAX_CHORD = 2 };

typedef struct {
  int32_t batch;   /* B ≥ 1                                                     */
  int32_t n;       /* variables, ≥ 1                                            */
  int32_t m_eq;    /* equality constraints, ≥ 0                         */
  int32_t p;       /* inequality constraints, ≥ 0                               */
  int64_t bstride_Q, bstride_q, bstride_A, bstride_b, bstride_G, bstride_h; /* elements; 0 = shared */
  /* A non-zero stride must be ≥ the per-problem size (n·n, n, m·n, m, p·n, p);
   * strides larger than that (padded batches) are accepted with
   * QP_MEM_DEVICE only — host modes take 0 or exactly the per-problem size
   * (QP_ERR_SHAPE otherwise). */
} qp_dims;

typedef struct {
  float tol;              /* relative residual + gap tolerance (Q4); default 1e-5          */
  int32_t max_iter;       /* Alg. 1 iterations; default 100                        */
  float sigma;            /* κ_target = σκ (Q2); default 0.1                        */
  float tau;              /* α = min(1, τ·α_max) (Eq. 6 + Q3); default 0.99                */
  float kappa_relax;      /* Alg. 2 target; default 1e-4                           */
  float relax_ktol;       /* |κ/κ_relax − 1| tolerance (Q5); default 1e-4                  */
  int32_t relax_max_iter; /* Alg. 2 iterations (Q22); default 50                           */
  int32_t formulation;    /* QP_IMPLICIT (default) | QP_EXPLICIT (config-3 standard arm)   */
  float pivot_floor_rel;  /* LDLᵀ pivot floor θ = rel·max|diag| (Q12); default √ε_f32     */
  int32_t mem_kind;       /* QP_MEM_DEVICE (default) | QP_MEM_HOST | QP_MEM_HOST_ASYNC     */
  float relax_tol;        /* Alg. 2 residual tolerance (Q5b); default 1e-6; the relax loop */
                          /* also stops at the f32 floor (φ ≤ tol and no 10% progress)     */
  int32_t relax_mode;     /* QP_RELAX_CHORD (default) | QP_RELAX_NEWTON (reading Q26, Q6) */
  int32_t chord_max;      /* QP_RELAX_CHORD: most chord steps per problem; default 8       */
  float chord_rho;        /* QP_RELAX_CHORD: contraction a chord step must reach, (0, 1];  */
                          /* default 0.5                                                    */
} qp_config;

typedef struct qp_ctx qp_ctx;

typedef struct {
  int32_t path;            /* 1-3: one CTA per QP for the whole call; KKT matrix in        */
                           /* 1 = shared memory, 2 = a global workspace (L2), 3 = shared   */
                           /* memory when the reduced system fits, else the workspace;     */
                           /* 4 = the batched phase engine (large shapes, the default for  */
                           /* everything path 1 cannot hold): one kernel per phase of a     */
                           /* Newton iteration over the whole batch, KKT matrices in        */
                           /* per-problem global workspaces, tensor-core assembly (one GEMM */
                           /* over the batch when G is shared) and Schur updates            */
  int32_t threads;         /* threads per CTA (path 4: of the per-problem phase kernels)   */
  int32_t smem_bytes;      /* dynamic shared memory per CTA (path 4: per-problem state)    */
  int32_t ctas_per_sm;     /* occupancy of the chosen kernel (path 4: 0, varies by phase)  */
  int32_t kkt_dim;         /* N = n4 + p + m (n4 = n rounded up to 4)                      */
  int32_t launches_solve;  /* kernel launches per qp_solve_batched (path 4: of the last    */
                           /* call — the count depends on the iterations it took)          */
  int32_t launches_backward;
  int64_t workspace_bytes;
  int32_t partition_cap;   /* largest number of constraints kept in augmented form in one */
                           /* reduced system (reading Q12c); p = no cap                    */
  int32_t handed_solve;    /* problems the last solve / backward handed to the uncapped    */
  int32_t handed_backward; /* large-N kernel (reading Q12c guard); synchronises the stream */
  int32_t relax_mode;      /* the Alg. 2 mode in effect (QP_RELAX_*)                       */
  int32_t chord_steps;     /* chord steps of the last backward, summed over the batch      */
                           /* (0 unless QP_RELAX_CHORD is in effect)                        */
} qp_info;

/* Fill *cfg with the defaults listed above. */
qp_err qp_config_default(qp_config* cfg);

/* Create a solver context for fixed dims/config on CUDA device `device`,
 * issuing work on `stream` (a cudaStream_t; NULL = legacy default stream).
 * Fails with QP_ERR_SHAPE if n+p+m exceeds what the kernels support
 * (qp_max_kkt_dim). */
qp_err qp_create(qp_ctx** ctx, const qp_dims* dims, const qp_config* cfg, int device, void* stream);
qp_err qp_set_stream(qp_ctx* ctx, void* stream);
qp_err qp_get_info(const qp_ctx* ctx, qp_info* info);
int32_t qp_max_kkt_dim(int32_t formulation);

/* Algorithm 1 on every problem: CVXOPT initialisation (Q11)
 * then Newton steps on the implicit partially condensed system Eq. 14
 * until the relative test of Q4 holds or max_iter.
 * Outputs (caller-owned, [B][·]): x[n], s[p], z[p], y[m]; iters = Newton
 * steps taken; status per problem (see enum).  x is Alg. 1's x* (κ → 0), not
 * the relaxed point (Q14). */
qp_err qp_solve_batched(qp_ctx* ctx, const float* Q, const float* q, const float* A, const float* b,
                        const float* G, const float* h, float* x, float* s, float* z, float* y,
                        int32_t* iters, int32_t* status);

/* Algorithm 2 (relax to κ_relax, exact Newton, factor-then-check: Q5, Q6)
 * followed by Algorithm 3: solve the bounded KKT system with
 * right-hand side (−∇ₓℓ, 0, 0) using the relaxed factorisation (Q7), dz =
 * d₊⊙dv (Q8), then ∇Q = ½(dx xᵀ + x dxᵀ), ∇q = dx, ∇A = dy xᵀ + y dxᵀ,
 * ∇b = −dy, ∇G = dz xᵀ + z dxᵀ, ∇h = −dz at the relaxed (x, y, z).
 * dl_dx: [B][n].  Gradient outputs have the batch layout of the matching
 * input: for a shared input (stride 0) the gradient is the BATCH SUM, a single
 * [n][n] / [n] / [m][n] / [m] / [p][n] / [p] array.  Any gradient pointer may be
 * NULL to skip it.  relax_iters/status: per problem (may be NULL). */
qp_err qp_backward_batched(qp_ctx* ctx, const float* dl_dx, float* dQ, float* dq, float* dA, float* db,
                           float* dG, float* dh, int32_t* relax_iters, int32_t* status);

/* Algorithmic flops executed by the LAST qp_solve_batched / qp_backward_batched
 * on this ctx, summed over the batch (the work model of DESIGN.md §6, counted
 * per problem inside the kernels from the actual iteration counts and reduced
 * system sizes).  Synchronises the ctx stream.  Either pointer may be NULL. */
qp_err qp_last_flops(qp_ctx* ctx, double* solve_flops, double* backward_flops);

qp_err qp_destroy(qp_ctx* ctx);

/* Diagnostic (tests only): dense H = Q + Gᵀ diag(om) G (n×n, row-major) on
 * the 3×TF32 tcgen05 tensor-core tile routine used by the large-n assembly.
 * All pointers device memory; asynchronous on `stream`. */
qp_err qp_debug_tc_syrk(const float* G, const float* om, const float* Q, int32_t n, int32_t p, float* H,
                        void* stream);
/* Diagnostic (tests only): with the environment variable QPB200_GUARD set at
 * qp_create, every ctx workspace is allocated with 64 KB guard bands of 0xFF
 * on both sides; this synchronises the ctx stream and counts the guard words
 * that no longer hold 0xFFFFFFFF (out-of-bounds writes by a kernel).
 * QP_ERR_UNSUPPORTED without guard mode. */
qp_err qp_debug_check_guards(qp_ctx* ctx, int64_t* bad_words);
const char* qp_error_string(qp_err err);

#ifdef __cplusplus
}
#endif
#endif /* QPB200_H */

// bnd_kernels.cuh — the BATCHED large-N engine (qp_info.path = 4): configs 4
// and 5 and every shape whose reduced KKT system does not fit a path-1 CTA.
//
// Why a second engine.  The persistent kernel of ipm_kernels.cuh runs one
// problem per CTA through the whole of Alg. 1 (or Alg. 2 + 3).  At config-4
// size (n = 200, p = 400, reduced systems of 300-540 rows) one CTA fills an
// SM, so each SM advances ONE problem through a chain of ~10⁴ dependent,
// barrier-separated steps per Newton iteration: the SM sits mostly idle on
// latency (round 1: 7.7 ms per problem, FP32 pipe < 10 %).  Here the same
// iteration is split into phases, each a kernel over the whole batch
// ("bulk-synchronous"), so that every SM holds several problems of every
// phase at once and the dependent chains of one problem hide behind those of
// the others:
//
//   bnd_begin                       CVXOPT initial system (solve) / load the
//                                   solution (backward)
//   per iteration k:
//     bnd_resid       (B CTAs)      v, κ, residuals Eq. 4 / Eq. 10, stop or
//                                   relax test, d±, c, ω, kept set, RHS
//     bnd_assemble    (tiles × B)   H = Q + Gᵀ diag(ω) G on tcgen05 (3×TF32)
//                                   tiles + the C / A rows and the diagonal
//     per 64-column panel c0:
//       bnd_tc_update (row tiles × B)  left-looking Schur update of the panel
//                                   on tcgen05 (3×TF32): K[i][c0:c1] −=
//                                   L[i][0:c0] S L[c0:c1][0:c0]ᵀ
//       bnd_pdiag     (B warps)     the panel's diagonal block: 16-wide
//                                   blocked signed Cholesky + inverses
//       bnd_prows     (row tiles × B)  the rows below it: per-thread
//                                   register forward substitution
//     bnd_solve       (B CTAs)      the two triangular solves (solve_qd)
//     bnd_update      (B CTAs)      Δv recovery, fraction-to-boundary step,
//                                   retraction — or, on the relaxed
//                                   iteration of the backward, Alg. 3
//
// Every phase calls the SAME device building blocks as the persistent kernel
// (residuals, compact_active, syrk_tile, tc_left_update, factor_big_range,
// invert_diag_block, solve_qd, recover_dv, newton_update, write_gradients),
// so the arithmetic of a Newton step is unchanged; only the schedule differs.
// Per-problem state (the iterate and the per-constraint vectors — the
// persistent kernel's shared-memory carve-up, Smem) lives in a global state
// block per problem, copied into shared memory by the phases that compute on
// it; the KKT matrix lives in a per-problem global workspace in the packed
// 16-row-block layout of ipm_cta.cuh.  DESIGN.md §5.
#pragma once
#include "ipm_kernels.cuh"
#include "kr_gemm.cuh"

namespace qpb {

enum { BM_DONE = 0, BM_INIT = 1, BM_NEWTON = 2, BM_ADJ = 3, BM_CHORD = 4 };

// Per-problem scalars: the first 16 words of every state block.
struct BScal {
  float kappa, kt, fl, phi_prev;
  float dmax;  // max |diag| of this iteration's KKT matrix (pivot floor θ = floor_rel·dmax)
  int mode, pa, it, status, ok;
  // guarded chord relax (reading Q26).  Solve: chord = 1 once this problem
  // cached a factorisation, cache_now = 1 on the iteration that does.
  // Backward: chord = 1 while chord steps are taken, nchord of them so far,
  // psi_prev = the previous ψ = max(φ, |κ/κ_relax − 1|).
  int chord, cache_now, nchord;
  float psi_prev;
  int pad[2];
};
static_assert(sizeof(BScal) == 64, "BScal: 16 words");

struct BArgs {
  Args a;               // problem data, outputs, settings (as for ipm_kernel)
  float* st;            // state blocks [B][st_stride]: BScal, then the Smem layout (no KKT buffer)
  long long st_stride;  // floats per state block (multiple of 4)
  float* kw;            // KKT workspaces [B][kstride] (packed layout of capacity Nmax)
  long long kstride;
  int* ctl;             // [0] problems still iterating after bnd_resid, [1] largest N4 among them
  int k;                // iteration index (bnd_resid)
  int c0, w;            // panel (bnd_tc_update, bnd_pdiag, bnd_prows)
  int ntiles;           // H tiles of the assembly (lower triangle of ⌈n4/128⌉² tiles; 0 = kr_gemm assembles H)
  // shared G (kr_gemm.cuh): this iteration's Ω rows (hi/lo tf32 split) of
  // the iterating problems by slot, and slot -> problem
  float *whi, *wlo;
  int* slotmap;
  int kr;
  float* dtg;           // [B][64·64]: the current panel's factored diagonal block, transposed (bnd_pdiag → bnd_prows)
  float* ug;            // [B][ustride]: the panel's Schur update U[i − c0][0:64] (bnd_tc_update → bnd_pdiag / bnd_prows)
  long long ustride;
  // TMA tensor maps of the KKT workspaces (bnd_tc_update_tma): one 128-byte
  // CUtensorMap per 16-row block b of the uniform packed layout, 3-D
  // {16b + 20 columns, 16 rows, problems}; this lane's first problem in them
  const char* tmaps;
  int lane_b0;
  // Q and G shared by the batch: the residual GEMVs as batched GEMMs
  // (bnd_sgemm): per problem Q x, Gᵀ z, Gᵀ t ([3][n4]); G x lands in the
  // state's gx segment.  nullptr = per-problem GEMVs inside bnd_resid
  float* pre;
  long long pre_stride;
  // forward substitution fused into the factorisation: bnd_pdiag solves the
  // panel's diagonal block for its rows of the right-hand side, bnd_prows
  // subtracts the panel's contribution from every row below, bnd_solve runs
  // only the backward substitution (chord steps: both)
  int fuse;
  int ntiles_tu;        // bnd_tc_update_tma: 128-row tiles of the panel in the lane's largest system
};

__device__ __forceinline__ float* st_of(const BArgs& b, int bid) { return b.st + (long long)bid * b.st_stride; }
__device__ __forceinline__ BScal& scal_of(float* st) { return *reinterpret_cast<BScal*>(st); }
__device__ __forceinline__ Smem carve_state(float* st, const Args& a) {
  return layout(st + 16, a.n4, a.m, a.p, a.N4max, 0, 0, 0);
}
__host__ inline long long bnd_state_floats(int n4, int m, int p, int N4max) {
  return (16 + (long long)(ipm_smem_bytes(n4, m, p, N4max, 0, 0, 0) / 4) + 3) & ~3LL;
}

// float4 copy of a state block (global ↔ shared), whole CTA, then a barrier
template <int NT>
__device__ __forceinline__ void copy_block(float* __restrict__ dst, const float* __restrict__ src, long long nf) {
  // 8 loads in flight per thread before the stores (the copy is latency-bound)
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  const int n4 = (int)(nf >> 2);
  for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * NT) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i0 + u * NT < n4) v[u] = s4[i0 + u * NT];
#pragma unroll
    for (int u = 0; u < 8; ++u) if (i0 + u * NT < n4) d4[i0 + u * NT] = v[u];
  }
  __syncthreads();
}

// The problem's KKT layout of this iteration: N = n4 + |kept| + m.
__device__ __forceinline__ KLayout bnd_layout(const Args& a, int pa) { return KLayout::make(a.n4 + pa + a.m, a.n4, true); }

// Solve finished (converged / failed / max_iter): outputs to the caller.
template <int NT>
__device__ void bnd_finish_solve(const Args& a, const Smem& S, BScal& h, int bid) {
  const int tid = threadIdx.x, n = a.n, m = a.m, p = a.p;
  for (int j = tid; j < n; j += NT) a.x[(long long)bid * n + j] = S.x[j];
  for (int l = tid; l < m; l += NT) a.y[(long long)bid * m + l] = S.y[l];
  for (int i = tid; i < p; i += NT) {
    a.z[(long long)bid * p + i] = S.z[i];
    a.s[(long long)bid * p + i] = S.s[i];
  }
  if (tid == 0) {
    a.iters[bid] = h.it;
    a.status[bid] = h.status;
    if (a.status_out) a.status_out[bid] = h.status;
    if (a.flops) a.flops[bid] = h.fl;
    h.mode = BM_DONE;
  }
}

// Backward finished: gradients (zero-filled unless h.ok) and counters.
template <int NT>
__device__ void bnd_finish_backward(const Args& a, const Smem& S, BScal& h, int bid) {
  const int tid = threadIdx.x, n = a.n, m = a.m, p = a.p;
  __syncthreads();
  if (!h.ok) {
    for (int j = tid; j < n; j += NT) { S.dx[j] = 0.f; S.x[j] = 0.f; }
    for (int l = tid; l < m; l += NT) { S.dy[l] = 0.f; S.y[l] = 0.f; }
    for (int i = tid; i < p; i += NT) { S.dz[i] = 0.f; S.z[i] = 0.f; }
    __syncthreads();
  }
  write_gradients<NT>(S, a, bid);
  if (tid == 0) {
    if (a.riters) a.riters[bid] = h.it;
    if (a.rstatus) a.rstatus[bid] = h.status;
    if (a.flops) a.flops[bid] = h.fl + 2.f * (n * n + m * n + p * n);
    h.mode = BM_DONE;
  }
}

// ---------------------------------------------------------------------------
// bnd_begin: solve — the CVXOPT initial system (reading Q11; the
// persistent kernel's iteration −1): ω = 1, nothing kept, right-hand side
// (−q + Gᵀh, b).  Backward — the solution of the last solve and its status.
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT) bnd_begin(const BArgs ba) {
  extern __shared__ __align__(16) float sm[];
  const Args& a = ba.a;
  const int bid = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, m = a.m, p = a.p;
  float* gst = st_of(ba, bid);
  const Smem S = carve_state(sm, a);
  BScal& h = scal_of(sm);
  const Prob P = prob_of(a, bid);
  if (tid == 0) {
    h.kappa = 0.f; h.kt = 0.f; h.fl = 0.f; h.phi_prev = INFINITY; h.dmax = 0.f;
    h.pa = 0; h.it = 0; h.status = ST_CONVERGED; h.ok = 0;
    h.cache_now = 0; h.nchord = 0; h.psi_prev = INFINITY;
    // solve: nothing cached yet; backward: chord steps iff the solve cached a factor
    h.chord = (a.bwd && a.kc && a.relax_mode == 2) ? a.chord_ok[bid] : 0;
    if (!a.bwd && a.chord_ok) a.chord_ok[bid] = 0;
  }
  if (!a.bwd) {
    for (int i = tid; i < p; i += NT) { S.om[i] = 1.f; S.v[i] = -1.f; }
    __syncthreads();
    compact_active<NT>(S, p, true, p);
    for (int j = tid; j < n4; j += NT) {
      float acc = 0.f;
      if (j < n) {
        acc = -__ldg(P.q + j);
        for (int i = 0; i < p; ++i) acc = fmaf(__ldg(P.G + i * n + j), __ldg(P.h + i), acc);
      }
      S.rhs[j] = acc;
    }
    for (int l = tid; l < m; l += NT) S.rhs[n4 + l] = __ldg(P.b + l);
    for (int j = n4 + m + tid; j < r4(n4 + m); j += NT) S.rhs[j] = 0.f;
    if (tid == 0) {
      h.mode = BM_INIT;
      h.fl = iter_flops(n, m, p, 0, false, true, true);
    }
    if (ba.kr) {  // Ω row of the initial system: ω = 1
      __shared__ int slot0;
      if (tid == 0) { slot0 = atomicAdd(ba.ctl, 1); ba.slotmap[slot0] = bid; }
      __syncthreads();
      kr::write_omega<NT>(ba.whi, ba.wlo, slot0, S.om, p, true);
    }
  } else {
    for (int j = tid; j < n; j += NT) S.x[j] = a.x[(long long)bid * n + j];
    for (int l = tid; l < m; l += NT) S.y[l] = a.y[(long long)bid * m + l];
    for (int i = tid; i < p; i += NT) {
      S.z[i] = a.z[(long long)bid * p + i];
      S.s[i] = a.s[(long long)bid * p + i];
    }
    const bool solved = (a.status[bid] & 0xff) == ST_CONVERGED;
    if (tid == 0) {
      h.mode = BM_NEWTON;  // bnd_resid decides
      if (!solved) h.status = ST_FAIL | (STG_RELAX << 8);
    }
    __syncthreads();
    if (!solved) bnd_finish_backward<NT>(a, S, h, bid);
  }
  __syncthreads();
  copy_block<NT>(gst, sm, ba.st_stride);
}

// ---------------------------------------------------------------------------
// bnd_resid (iteration k ≥ 0): manifold coordinates, residuals and the
// stopping test (solve: Q4; backward: the relax test Q5/Q5b), then the data
// of this iteration's Newton system — exactly the head of the persistent
// kernel's loop body.
// ---------------------------------------------------------------------------
template <int NT, bool LARGE = false>
__global__ void __launch_bounds__(NT) bnd_resid(const BArgs ba) {
  extern __shared__ __align__(16) float sm[];
  const Args& a = ba.a;
  const int bid = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, m = a.m, p = a.p;
  float* gst = st_of(ba, bid);
  if (scal_of(gst).mode == BM_DONE) return;
  copy_block<NT>(sm, gst, ba.st_stride);
  const Smem S = carve_state(sm, a);
  BScal& h = scal_of(sm);
  const Prob P = prob_of(a, bid);
  const bool bwd = a.bwd != 0;
  const int k = ba.k;
  const float kappa = manifold_coords<NT>(S, a);
  const float kt = bwd ? a.kappa_relax : a.sigma * kappa;
  // guarded chord relax (reading Q26): a problem in chord mode computes its
  // residuals with the cached Jacobian (the right-hand side of the chord step)
  const bool was_chord = bwd && h.chord;
  const float* cj = was_chord ? a.chd + (long long)bid * a.chd_stride : nullptr;
  if (was_chord) {
    const int p4 = (p + 3) & ~3;
    for (int i = tid; i < p; i += NT) {
      S.dp[i] = cj[4 + i]; S.dm[i] = cj[4 + p4 + i]; S.c[i] = cj[4 + 2 * p4 + i];
      S.widx[i] = __float_as_int(cj[4 + 3 * p4 + i]);
    }
    __syncthreads();
  }
  // One call site for both passes (a second pass recomputes the current
  // Jacobian when a chord phase ends): a single inlined copy of residuals(),
  // so a problem that leaves chord mode computes exactly what exact Newton does.
  Norms R;
  bool fin = false, adj = false, chord = was_chord, cache = false, keep = was_chord;
  int status = ST_CONVERGED, nchord = h.nchord;
  float fl = h.fl, phi_prev = h.phi_prev, psi_prev = h.psi_prev;
#pragma unroll 1
  for (int pass = 0;; ++pass) {
    R = residuals<NT, LARGE>(S, a, P, kappa, kappa - kt, keep, keep ? __float_as_int(cj[0]) : 0,
                             ba.pre ? ba.pre + (long long)bid * ba.pre_stride : nullptr);
    if (pass == 1) break;
    if (R.nonfin > 0.f) {
      status = ST_FAIL | ((bwd ? STG_RELAX : STG_SCALING) << 8);
      fin = true;
    } else if (!bwd) {
      if (converged_solve(R, a.tol)) {
        fl += iter_flops(n, m, p, 0, true, false, false);
        fin = true;
      } else if (k == a.max_iter) {
        fl += iter_flops(n, m, p, 0, true, false, false);
        status = ST_MAX_ITER;
        fin = true;
      } else if (a.kc && a.relax_mode == 2 && !h.chord && kappa < sqrtf(10.f) * a.kappa_relax) {
        cache = true;  // this iteration's factorisation is the one Alg. 2 will reuse
      }
    } else {
      const bool kok = p == 0 || fabsf(kappa / a.kappa_relax - 1.f) <= a.relax_ktol;
      if (chord) {  // the guard: chord steps while each shrinks ψ by chord_rho, at most chord_max
        const float psi = fmaxf(rel_phi(R), p == 0 ? 0.f : fabsf(kappa / a.kappa_relax - 1.f));
        if (nchord >= a.chord_max || (nchord > 0 && !(psi <= a.chord_rho * psi_prev))) {
          chord = false;
          phi_prev = INFINITY;  // the stall test (Q5b) measures Newton steps only
        }
        psi_prev = psi;
      }
      // a chord stops only at φ ≤ relax_tol (a slow chord is not the f32 floor)
      adj = kok && (chord ? rel_phi(R) <= a.relax_tol : relax_done(R, a.tol, a.relax_tol, phi_prev));
      phi_prev = kok ? rel_phi(R) : INFINITY;
      if (!adj && k == a.relax_max_iter) {
        status = ST_MAX_ITER | (STG_RELAX << 8);
        fin = true;
      }
    }
    // leaving chord mode: this iteration factors, with the Jacobian of the current point
    if (!(was_chord && !fin && (adj || !chord))) break;
    keep = false;
    __syncthreads();
  }
  if (adj || fin) chord = false;
  __syncthreads();
  if (tid == 0) {
    h.it = k; h.status = status; h.fl = fl; h.phi_prev = phi_prev;
    h.kappa = kappa; h.kt = kt; h.pa = R.pa; h.dmax = 0.f; h.ok = 0;
    h.psi_prev = psi_prev; h.cache_now = cache ? 1 : 0;
    if (bwd) h.chord = chord ? 1 : 0;
    else if (cache) h.chord = 1;
  }
  if (fin) {
    __syncthreads();
    if (!bwd) bnd_finish_solve<NT>(a, S, h, bid);
    else bnd_finish_backward<NT>(a, S, h, bid);
  } else if (chord) {  // a chord step: no assembly, no factorisation (reading Q26)
    if (tid == 0) {
      h.mode = BM_CHORD;
      h.nchord = nchord + 1;
      h.fl = fl + iter_flops(n, m, p, R.pa, true, false, true);
      atomicAdd(ba.ctl + 2, 1);
    }
  } else {
    if (adj)  // Algorithm 3: the relaxed system with right-hand side (−∇ₓℓ, 0, 0)
      for (int j = tid; j < a.N4max; j += NT) S.rhs[j] = j < n ? -__ldg(a.dl + (long long)bid * n + j) : 0.f;
    __shared__ int slot;
    if (tid == 0) {
      h.mode = adj ? BM_ADJ : BM_NEWTON;
      h.fl = fl + iter_flops(n, m, p, R.pa, true, true, true);
      slot = atomicAdd(ba.ctl, 1);
      atomicMax(ba.ctl + 1, r4(n4 + R.pa + m));
      if (cache) atomicAdd(ba.ctl + 3, 1);
      if (ba.kr) ba.slotmap[slot] = bid;
    }
    if (ba.kr) {  // this problem's Ω row for the batched assembly GEMM
      __syncthreads();
      kr::write_omega<NT>(ba.whi, ba.wlo, slot, S.om, p, false);
    }
  }
  __syncthreads();
  copy_block<NT>(gst, sm, ba.st_stride);
}

// ---------------------------------------------------------------------------
// bnd_scatter: grid B — the rows ≥ n4 of the KKT matrix (zeroed, then the
// kept C rows d₊ₖ gₖ, the A rows, the diagonal −d₋ / 0 / −1) when H comes
// from kr_gemm (shared G); bnd_assemble's last CTA does the same otherwise.
// ---------------------------------------------------------------------------

// One warp per row r ≥ n4 (bnd_scatter, and bnd_assemble's last CTA), each element written once
// (columns < n: the C / A row or zeros on padding rows; columns n .. len:
// zeros, float4 from n4; then the diagonal), instead of zeroing the whole
// tail of the workspace and writing the C / A rows over it
template <int NT>
__device__ __forceinline__ void scatter_rows_once(const Args& a, const Smem& S, const KLayout& L, float* K,
                                                  const Prob& P, int pa, float& dmax) {
  const int tid = threadIdx.x, lane = tid & 31, n = a.n, n4 = a.n4, N = L.N, N4 = L.N4;
  for (int r = n4 + (tid >> 5); r < N4; r += NT / 32) {
    const int rr = r - n4;
    const float* src = nullptr;
    float w = 1.f, d;
    if (rr < pa) {
      const int kk = S.act[rr];
      src = P.G + (size_t)kk * n;
      w = S.dp[kk];
      const float e = S.dm[kk];
      d = -e;
      dmax = fmaxf(dmax, fabsf(e));
    } else if (r < N) {
      src = P.A + (size_t)(rr - pa) * n;
      d = 0.f;
    } else {
      d = -1.f;
    }
    float* dst = K + L.off(r);
    const int len = L.len(r >> 4);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int q = (n4 >> 2) + lane; q < (len >> 2); q += 32) d4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (src && !(n & 3) && !(reinterpret_cast<uintptr_t>(src) & 15)) {  // float4 row copy
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int q = lane; q < (n >> 2); q += 32) {
        const float4 v = __ldg(s4 + q);
        d4[q] = make_float4(w * v.x, w * v.y, w * v.z, w * v.w);
      }
    } else if (src) {
      for (int j = lane; j < n; j += 32) dst[j] = w * __ldg(src + j);
    } else {
      for (int j = lane; j < n; j += 32) dst[j] = 0.f;
    }
    for (int j = n + lane; j < n4; j += 32) dst[j] = 0.f;
    __syncwarp();
    if (lane == 0) dst[r] = d;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) bnd_scatter(const BArgs ba) {
  const Args& a = ba.a;
  const int bid = blockIdx.x;
  float* gst = st_of(ba, bid);
  BScal& h = scal_of(gst);
  if (h.mode == BM_DONE || h.mode == BM_CHORD) return;
  const int pa = h.pa;
  const KLayout L = bnd_layout(a, pa);
  float dmax = 0.f;
  if (ba.pre && h.mode == BM_NEWTON) {  // + Gᵀ t of the batched GEMM, before the fused forward substitution
    float* rhs = carve_state(gst, a).rhs;
    const float* gt = ba.pre + (long long)bid * ba.pre_stride + 2 * a.n4;
    for (int j = threadIdx.x; j < a.n; j += NT) rhs[j] += gt[j];
  }
  scatter_rows_once<NT>(a, carve_state(gst, a), L, ba.kw + (long long)bid * ba.kstride, prob_of(a, bid), pa, dmax);
#pragma unroll
  for (int o = 16; o; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((threadIdx.x & 31) == 0 && dmax > 0.f) atomicMax(reinterpret_cast<int*>(&h.dmax), __float_as_int(dmax));
}

// ---------------------------------------------------------------------------
// bnd_assemble: grid (ntiles + 1, B).  CTA x < ntiles: one 128×128 tile of
// H = Q + Gᵀ diag(ω) G (tcgen05, 3×TF32; tc_syrk.cuh), lower triangle, the
// epilogue adding Q (identity on the padding rows n..n4).  CTA x = ntiles:
// the rows ≥ n4 — zeroed, then the kept C rows d₊ₖ gₖ, the A rows and the
// diagonal (−d₋ on the kept rows, 0 for y, −1 on padding).  Both record
// max|diag| (θ of the pivot floor) with an atomic max.
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT) bnd_assemble(const BArgs ba) {
  extern __shared__ __align__(128) float smtc[];
  float* sm = smtc;
  const Args& a = ba.a;
  const int bid = blockIdx.y, tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p;
  float* gst = st_of(ba, bid);
  BScal& h = scal_of(gst);
  if (h.mode == BM_DONE || h.mode == BM_CHORD) return;
  const Smem S = carve_state(gst, a);  // global state (read only here)
  const int pa = h.pa;
  const KLayout L = bnd_layout(a, pa);
  float* K = ba.kw + (long long)bid * ba.kstride;
  const Prob P = prob_of(a, bid);
  const int N = L.N, N4 = L.N4;
  float dmax = 0.f;
  if ((int)blockIdx.x == ba.ntiles) {
    scatter_rows_once<NT>(a, S, L, K, P, pa, dmax);
  } else {
    int I = 0, t = blockIdx.x;
    while (t > I) { t -= I + 1; ++I; }
    const int i0 = tc::TM * I, j0 = tc::TN * t;
    const tc::TcState ts = tc::tc_state(sm);
    tc::tmem_alloc(ts);
    tc::syrk_tile<NT>(ts, P.G, S.om, p, n, i0, j0, [&](int row0, int j, const float* tt) {
      float qv[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int i = row0 + r;
        qv[r] = (i < n && j < n && j <= i) ? __ldg(P.Q + (size_t)i * n + j) : 0.f;
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int i = row0 + r;
        if (i < n4 && j <= i) {
          const float val = (i < n && j < n) ? qv[r] + tt[33 * r] : (i == j ? 1.f : 0.f);
          K[L.off(i) + j] = val;
          if (i == j && i < n) dmax = fmaxf(dmax, fabsf(val));
        }
      }
    });
    tc::tmem_free(*ts.tmem_slot);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  if ((tid & 31) == 0 && dmax > 0.f) atomicMax(reinterpret_cast<int*>(&h.dmax), __float_as_int(dmax));
}

// ---------------------------------------------------------------------------
// bnd_tc_update: grid (row tiles, B), panel [c0, c0 + 64), c0 > 0: for rows
// [c0 + 128·x, +128) the Schur update of the panel from every earlier column
//     U[i][c] = Σ_{k<c0} L[i][k] S_k L[c0+c][k]
// on tcgen05 (3×TF32 split, TMEM accumulator 128 × 64): each thread stages
// 12 fixed 16-byte row pieces per 32-deep K chunk (row offsets computed
// once) in registers, the next chunk's loads in flight while the MMAs of
// this one run.  The result goes to the per-problem buffer U (each thread
// writes its TMEM lane's 32-column row segments); bnd_pdiag / bnd_prows
// subtract it when they load the panel — K itself is read here only as the
// operands, never read-modified-written.
// ---------------------------------------------------------------------------
#ifndef QPB200_TCU_PREF
#define QPB200_TCU_PREF 5  // bnd_tc_update: L2 prefetch distance in K chunks (3: −0.5 %, 2: −0.4 %)
#endif
template <int NT>
__global__ void __launch_bounds__(NT, 3) bnd_tc_update(const BArgs ba) {
  static_assert(NT == 128, "bnd_tc_update: 128 threads (16 rows x 8 K-quads per pass)");
  using tc::TK;
  constexpr int TM = 128, BW = 64, SA = TM / 16, SB = BW / 16;  // row passes of A and B per thread
  extern __shared__ __align__(128) float smtc[];
  const Args& a = ba.a;
  const int bid = blockIdx.y, tid = threadIdx.x;
  const BScal& h = scal_of(st_of(ba, bid));
  if (h.mode == BM_DONE || h.mode == BM_CHORD) return;
  const KLayout L = bnd_layout(a, h.pa);
  const int c0 = ba.c0, i0 = c0 + TM * (int)blockIdx.x, N4 = L.N4, npos = L.npos;
  if (c0 >= N4 || i0 >= N4) return;
  const int c1 = min(c0 + BW, N4), wn = (c1 - c0 + 15) & ~15;
  const float* K = ba.kw + (long long)bid * ba.kstride;
  const tc::TcState ts = tc::tc_state(smtc);
  tc::tmem_alloc(ts);
  const uint32_t tmem = *ts.tmem_slot;
  uint32_t phase = *ts.phase_slot;
  const uint32_t idesc = tc_idesc_n(wn);
  // thread → (row, K quad): lanes 8h..8h+7 take rows 8·warp + [0, 8) at quad h (+4): a
  // quarter-warp stores one core-matrix column of 8 rows (conflict-free) and
  // the four quarter-warps read 64 contiguous bytes of each row (whole sectors)
  const int warp = tid >> 5, lane = tid & 31, rl8 = lane & 7, qq = lane >> 3;
  int ro[SA / 2 + SB / 2];  // rows 8·warp + rl8 + 32·s: A s < 4, B s < 2
#pragma unroll
  for (int s2 = 0; s2 < SA / 2; ++s2) { const int i = i0 + 8 * warp + rl8 + 32 * s2; ro[s2] = i < N4 ? L.off(i) : -1; }
#pragma unroll
  for (int s2 = 0; s2 < SB / 2; ++s2) { const int j = c0 + 8 * warp + rl8 + 32 * s2; ro[SA / 2 + s2] = j < c1 ? L.off(j) : -1; }
  float4 rg[SA + SB];  // [2 quads][rows]: index h·(SA/2 + SB/2) + s
  constexpr int NR = SA / 2 + SB / 2;
  auto load = [&](int k0) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int k = k0 + 4 * (qq + 4 * h2);
#pragma unroll
      for (int s2 = 0; s2 < NR; ++s2)
        rg[h2 * NR + s2] = (ro[s2] >= 0 && k < c0) ? *reinterpret_cast<const float4*>(K + ro[s2] + k)
                                                    : make_float4(0, 0, 0, 0);
    }
  };
  // L2 prefetch of a later chunk's pieces (the register stage is one chunk
  // ahead; the A rows of the panel update come from HBM)
  auto pref = [&](int k0) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int k = k0 + 4 * (qq + 4 * h2);
#pragma unroll
      for (int s2 = 0; s2 < NR; ++s2)
        if (ro[s2] >= 0 && k < c0) asm volatile("prefetch.global.L2 [%0];" ::"l"(K + ro[s2] + k));
    }
  };
  auto split4 = [](float4 v, float4& hi, float4& lo) {
    hi.x = tc::to_tf32(v.x); lo.x = tc::to_tf32(v.x - hi.x);
    hi.y = tc::to_tf32(v.y); lo.y = tc::to_tf32(v.y - hi.y);
    hi.z = tc::to_tf32(v.z); lo.z = tc::to_tf32(v.z - hi.z);
    hi.w = tc::to_tf32(v.w); lo.w = tc::to_tf32(v.w - hi.w);
  };
  load(0);
  for (int k0 = 0; k0 < c0; k0 += TK) {
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int qd = qq + 4 * h2;
      const bool neg = k0 + 4 * qd >= npos;  // S_k on the B operand (npos is a multiple of 4)
#pragma unroll
      for (int s2 = 0; s2 < NR; ++s2) {
        float4 v = rg[h2 * NR + s2], hi, lo;
        const bool isb = s2 >= SA / 2;
        if (isb && neg) { v.x = -v.x; v.y = -v.y; v.z = -v.z; v.w = -v.w; }
        split4(v, hi, lo);
        const int sr = isb ? s2 - SA / 2 : s2;
        const int o = ((warp + 4 * sr) * (TK / 4) + qd) * 32 + rl8 * 4;  // canonical K-major (op_offset)
        *reinterpret_cast<float4*>((isb ? ts.bhi : ts.ahi) + o) = hi;
        *reinterpret_cast<float4*>((isb ? ts.blo : ts.alo) + o) = lo;
      }
    }
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::tc_fence_after();
      const uint32_t ahi = tc::smem_u32(ts.ahi), alo = tc::smem_u32(ts.alo);
      const uint32_t bhi = tc::smem_u32(ts.bhi), blo = tc::smem_u32(ts.blo);
#pragma unroll
      for (int ks = 0; ks < TK / 8; ++ks) {
        const uint32_t off = ks * 2 * 128;
        const uint32_t acc0 = (k0 > 0 || ks > 0) ? 1u : 0u;
        tc::mma_tf32(tmem, tc::make_desc(ahi + off), tc::make_desc(bhi + off), idesc, acc0);
        tc::mma_tf32(tmem, tc::make_desc(ahi + off), tc::make_desc(blo + off), idesc, 1u);
        tc::mma_tf32(tmem, tc::make_desc(alo + off), tc::make_desc(bhi + off), idesc, 1u);
      }
      tc::commit(ts.mbar);
    }
    if (k0 + TK < c0) load(k0 + TK);  // in flight while the MMAs run
    if (k0 + QPB200_TCU_PREF * TK < c0) pref(k0 + QPB200_TCU_PREF * TK);
    tc::mbar_wait(ts.mbar, phase);
    phase ^= 1u;
    tc::tc_fence_after();
  }
  // epilogue: TMEM lane = row i0 + 32·warp + lane → registers → per-warp
  // transpose (the operand tiles are idle now) → coalesced 128-byte rows of U
  float* T = ts.ahi + warp * (32 * 33);
  float* U = ba.ug + (long long)bid * ba.ustride;
  for (int cc = 0; cc < wn; cc += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)cc, v);
#pragma unroll
    for (int c = 0; c < 32; ++c) T[lane * 33 + c] = v[c];
    __syncwarp();
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      const int i = i0 + 32 * warp + r;
      if (i < N4) U[(long long)(i - c0) * BW + cc + lane] = T[r * 33 + lane];
    }
    __syncwarp();
  }
  tc::tmem_free(tmem);
}

// ---------------------------------------------------------------------------
// bnd_tc_update_tma: the same Schur update of a panel as bnd_tc_update, its
// operands staged by the Tensor Memory Accelerator.  Per 32-deep K chunk one
// thread issues 3-D tensor copies (cp.async.bulk.tensor, one per 16-row
// block: A = rows [i0, i0 + 128), B = rows [c0, c0 + 64), columns [k0, k0 +
// 32)) into an S-stage ring of fp32 tiles in the 128-byte-swizzled K-major
// layout (a row's 128 bytes, 16-byte chunks XOR-permuted by row mod 8),
// completing on the stage's mbarrier.  The CTA splits a landed chunk IN
// PLACE for 3×TF32 — hi = tf32(x) over x, lo = tf32(x − hi) into the stage's
// lo tiles, the sign S_k applied to B — and one thread issues the 12 MMAs
// reading the swizzled tiles directly (SWIZZLE_128B descriptors).  Because
// every stage carries its own operands, the split of chunk k + 1 overlaps
// the MMAs of chunk k, and a stage is refilled (chunk k − 1 + S) once its
// MMAs have completed (tcgen05.commit on the stage's second mbarrier).  The
// ring hides the HBM latency that bounds the register-staged kernel
// (profiles/r2: 36 % of its stall samples wait on those loads).
// ---------------------------------------------------------------------------
namespace tu {
constexpr int TM = 128, BW = 64, TK = 32;
constexpr int TA = TM * TK * 4, TB = BW * TK * 4;  // 16 KB, 8 KB
constexpr int RAW = TA + TB;                        // a TMA stage: raw A, raw B
constexpr int OPS = 2 * (TA + TB);                  // an operand buffer: hi A, hi B, lo A, lo B
__host__ __device__ constexpr int smem_bytes(int S, int NOB = 2) { return 1024 + S * RAW + NOB * OPS + 256; }

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* map, int c0, int c1, int c2, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
// K-major SWIZZLE_128B operand: 8-row groups 1024 B apart (SBO); the K step
// inside the 128-byte swizzle atom advances the start address (32 B per 8 tf32)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused by swizzled K-major layouts)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;              // version (sm_100)
  d |= (uint64_t)2 << 61;              // layout: SWIZZLE_128B
  return d;
}
}  // namespace tu

// Persistent and warp-specialised (448 threads, one CTA per SM): work items
// are (problem, 128-row tile) pairs of the panel, strided over the grid
// (tile fastest); every role walks the same item sequence.
//   warp 8      producer: TMA copies of item j's K chunk into raw stage j % S
//   warps 0-7   split: raw stage → 3×TF32 hi/lo operand buffer j % 2 (SW128);
//               warp w takes rows 8·(w % 4) + 32·t + [0, 8) at K quads
//               4·(w / 4) + [0, 4)
//   warp 9      MMA issuer: 12 tcgen05.mma per chunk into one of TWO TMEM
//               accumulators (one per tile, alternating)
//   warps 10-13 epilogue: the other accumulator → U (TMEM lane quarter w % 4)
// mbarriers: full / rawfree per raw stage, opfull / opfree per operand
// buffer, accfull / accfree per accumulator.
constexpr int TU_THREADS = 448;
constexpr int TU_SPLIT = 8;  // split warps

template <int S, int NOB>
__global__ void __launch_bounds__(TU_THREADS, 1) bnd_tc_update_tma(const BArgs ba) {
  using namespace tu;
  constexpr int SA = TM / 32, SB = BW / 32;  // 32-row groups of A and B per split thread
  extern __shared__ unsigned char smdyn[];
  const Args& a = ba.a;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c0 = ba.c0, nk = c0 / TK;  // c0 is a multiple of 64
  const int T = ba.ntiles_tu;          // row tiles of the largest problem of the lane
  const long long nq = (long long)ba.a.B * T;
  // the work-item walk shared by every role: q = blockIdx.x + g·gridDim.x,
  // problem q / T, tile q % T, skipped unless the problem factors and has that tile
  struct Item { int y, i0, N4, npos; };
  auto valid = [&](long long q, Item& it) {
    const int y = (int)(q / T), t = (int)(q % T);
    const BScal& h = scal_of(st_of(ba, y));
    if (h.mode == BM_DONE || h.mode == BM_CHORD) return false;
    const KLayout L = bnd_layout(a, h.pa);
    const int i0 = c0 + TM * t;
    if (c0 >= L.N4 || i0 >= L.N4) return false;
    it.y = y; it.i0 = i0; it.N4 = L.N4; it.npos = L.npos;
    return true;
  };
  auto next = [&](long long& q, Item& it) {  // advance to the next valid item (q < 0: start)
    q = q < 0 ? (long long)blockIdx.x : q + gridDim.x;
    while (q < nq && !valid(q, it)) q += gridDim.x;
    return q < nq;
  };
  const uint32_t base_s = (tc::smem_u32(smdyn) + 1023u) & ~1023u;
  unsigned char* base = smdyn + (base_s - tc::smem_u32(smdyn));
  unsigned char* opb = base + S * RAW;
  uint64_t* full = reinterpret_cast<uint64_t*>(opb + NOB * OPS);
  uint64_t* rawfree = full + S;
  uint64_t* opfull = rawfree + S;
  uint64_t* opfree = opfull + NOB;
  uint64_t* accfull = opfree + NOB;
  uint64_t* accfree = accfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accfree + 2);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(tc::smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int st = 0; st < S; ++st) { tc::mbar_init(full + st, 1); tc::mbar_init(rawfree + st, TU_SPLIT); }
    for (int b = 0; b < NOB; ++b) { tc::mbar_init(opfull + b, TU_SPLIT); tc::mbar_init(opfree + b, 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(accfull + b, 1); tc::mbar_init(accfree + b, 4); }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == TU_SPLIT) {
    if (lane == 0) {  // producer
      long long q = -1;
      Item it;
      int j = 0;
      while (next(q, it)) {
        const int bA = it.i0 >> 4, bB = c0 >> 4, c1 = min(c0 + BW, it.N4);
        int nA = 0, nB = 0;
        for (int t = 0; t < SA * 2; ++t) nA += (16 * (bA + t) < it.N4) ? 1 : 0;
        for (int t = 0; t < SB * 2; ++t) nB += (16 * (bB + t) < c1) ? 1 : 0;
        const int prob = ba.lane_b0 + it.y;
        for (int kc = 0; kc < nk; ++kc, ++j) {
          const int st = j % S;
          if (j >= S) tc::mbar_wait(rawfree + st, (uint32_t)(((j / S) - 1) & 1));
          const uint32_t mb = tc::smem_u32(full + st);
          expect_tx(mb, (uint32_t)(nA + nB) * 2048u);
          const uint32_t dA = base_s + st * RAW, dB = dA + TA;
          for (int t = 0; t < nA; ++t) tma_load_3d(dA + t * 2048, ba.tmaps + (size_t)(bA + t) * 128, TK * kc, 0, prob, mb);
          for (int t = 0; t < nB; ++t) tma_load_3d(dB + t * 2048, ba.tmaps + (size_t)(bB + t) * 128, TK * kc, 0, prob, mb);
        }
      }
    }
  } else if (warp == TU_SPLIT + 1) {
    if (lane == 0) {  // MMA issuer
      long long q = -1;
      Item it;
      int j = 0, u = 0;
      while (next(q, it)) {
        const int acc = u & 1;
        const int c1 = min(c0 + BW, it.N4), wn = (c1 - c0 + 15) & ~15;
        const uint32_t idesc = tc_idesc_n(wn), tacc = tmem + (uint32_t)(acc * BW);
        if (u >= 2) tc::mbar_wait(accfree + acc, (uint32_t)(((u >> 1) - 1) & 1));  // drained by the epilogue
        tc::tc_fence_after();
        for (int kc = 0; kc < nk; ++kc, ++j) {
          const int b = j % NOB;
          tc::mbar_wait(opfull + b, (uint32_t)((j / NOB) & 1));
          tc::tc_fence_after();
          const uint32_t uhA = base_s + S * RAW + b * OPS, uhB = uhA + TA, ulA = uhB + TB, ulB = ulA + TA;
#pragma unroll
          for (int ks = 0; ks < TK / 8; ++ks) {
            const uint32_t off = ks * 32;  // 8 tf32 of K in the 128-byte swizzle atom
            const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
            tc::mma_tf32(tacc, desc_sw128(uhA + off), desc_sw128(uhB + off), idesc, acc0);
            tc::mma_tf32(tacc, desc_sw128(uhA + off), desc_sw128(ulB + off), idesc, 1u);
            tc::mma_tf32(tacc, desc_sw128(ulA + off), desc_sw128(uhB + off), idesc, 1u);
          }
          tc::commit(opfree + b);
        }
        tc::commit(accfull + acc);
        ++u;
      }
    }
  } else if (warp < TU_SPLIT) {
    // split: a quarter-warp takes rows 8·w4 + [0, 8) at one K quad (8 distinct
    // swizzled 16-byte chunks: conflict-free); rows past N4 / c1 become zeros
    const int rl8 = lane & 7, qq = (lane >> 3) + 4 * (warp >> 2), w4 = warp & 3;
    long long q = -1;
    Item it;
    int j = 0;
    while (next(q, it)) {
      const int c1 = min(c0 + BW, it.N4);
      for (int kc = 0; kc < nk; ++kc, ++j) {
        const int st = j % S, b = j % NOB, k0 = TK * kc;
        const float* rA = reinterpret_cast<const float*>(base + st * RAW);
        const float* rB = rA + TA / 4;
        float* hA = reinterpret_cast<float*>(opb + b * OPS);
        float* hB = hA + TA / 4;
        float* lA = hB + TB / 4;
        float* lB = lA + TA / 4;
        tc::mbar_wait(full + st, (uint32_t)((j / S) & 1));
        if (j >= NOB) tc::mbar_wait(opfree + b, (uint32_t)(((j / NOB) - 1) & 1));  // the MMAs of item j − NOB read it
        float4 v[1][SA + SB];
        {
          const int sw = (qq ^ rl8) << 2;
#pragma unroll
          for (int s2 = 0; s2 < SA + SB; ++s2) {
            const bool isb = s2 >= SA;
            const int r = 8 * w4 + rl8 + 32 * (isb ? s2 - SA : s2);
            v[0][s2] = *reinterpret_cast<const float4*>((isb ? rB : rA) + r * TK + sw);
          }
        }
        __syncwarp();
        if (lane == 0) kr::mbar_arrive(rawfree + st);  // this warp has read the raw stage
        {
          const int h2 = 0, qd = qq;
          const bool neg = k0 + 4 * qd >= it.npos;  // S_k on the B operand (npos is a multiple of 4)
          const int sw = (qd ^ rl8) << 2;
#pragma unroll
          for (int s2 = 0; s2 < SA + SB; ++s2) {
            const bool isb = s2 >= SA;
            const int r = 8 * w4 + rl8 + 32 * (isb ? s2 - SA : s2);
            const bool ok = isb ? c0 + r < c1 : it.i0 + r < it.N4;
            float4 x = ok ? v[h2][s2] : make_float4(0.f, 0.f, 0.f, 0.f), hi, lo;
            if (isb && neg) { x.x = -x.x; x.y = -x.y; x.z = -x.z; x.w = -x.w; }
            hi.x = tc::to_tf32(x.x); lo.x = tc::to_tf32(x.x - hi.x);
            hi.y = tc::to_tf32(x.y); lo.y = tc::to_tf32(x.y - hi.y);
            hi.z = tc::to_tf32(x.z); lo.z = tc::to_tf32(x.z - hi.z);
            hi.w = tc::to_tf32(x.w); lo.w = tc::to_tf32(x.w - hi.w);
            *reinterpret_cast<float4*>((isb ? hB : hA) + r * TK + sw) = hi;
            *reinterpret_cast<float4*>((isb ? lB : lA) + r * TK + sw) = lo;
          }
        }
        tc::fence_async_smem();
        __syncwarp();
        if (lane == 0) kr::mbar_arrive(opfull + b);
      }
    }
  } else {
    // epilogue warps 10-13: TMEM lane quarter g = warp % 4 → rows i0 + 32g + lane of U
    const int g = warp & 3;
    long long q = -1;
    Item it;
    int u = 0;
    while (next(q, it)) {
      const int acc = u & 1;
      const int c1 = min(c0 + BW, it.N4), wn = (c1 - c0 + 15) & ~15;
      tc::mbar_wait(accfull + acc, (uint32_t)((u >> 1) & 1));
      tc::tc_fence_after();
      const int i = it.i0 + 32 * g + lane;
      float* U = ba.ug + (long long)it.y * ba.ustride;
      for (int cc = 0; cc < wn; cc += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * g) << 16) + (uint32_t)(acc * BW + cc), v);
        if (i < it.N4) {
          float4* dst = reinterpret_cast<float4*>(U + (long long)(i - c0) * BW + cc);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4) dst[q4] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) kr::mbar_arrive(accfree + acc);
      ++u;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// The panel [c0, c0 + w) (w = 64 except the last panel) after its Schur
// update, in two kernels:
//   bnd_pdiag (grid B, ONE warp per problem): the w×w diagonal block in
//     shared memory, factored (factor_big_range on a dense PanelLayout:
//     16×16 diagonal blocks with a register window, TRSM, update; pivot floor
//     θ = floor_rel·max|diag|, reading Q12), its 16×16 diagonal-block
//     inverses W_b formed (for solve_qd) and the block written back.  The
//     pivot chain of a panel is inherently serial; one warp per problem keeps
//     up to 12 such chains in flight per SM instead of one per 128 threads.
//   bnd_prows (grid (128-row tiles, B)): every row i below the block finished
//     by ONE thread in registers — forward substitution of its 64 panel
//     entries against the factored block, x_k = a_k / L_kk, a_j −= x_k L_jk
//     (j > k), stored L_ik = S_k x_k: the TRSM and the in-panel Schur updates
//     of all four 16-column blocks in one pass over the row.
// ---------------------------------------------------------------------------
#ifndef QPB200_PDIAG_QS
#define QPB200_PDIAG_QS 4  // bnd_pdiag trailing-update rows per pass (ipm_cta.cuh factor_big_range)
#endif
namespace pnl {
constexpr int W = 64, DS = 68;  // panel width, dense row stride (odd multiple of 16 B)
}

template <int NT>
__global__ void __launch_bounds__(NT) bnd_pdiag(const BArgs ba) {
  using namespace pnl;
  __shared__ __align__(16) float D[W * DS];
  __shared__ float scr[16 * 17 + 16];
  const Args& a = ba.a;
  const int bid = blockIdx.x, tid = threadIdx.x;
  float* gst = st_of(ba, bid);
  const BScal& h = scal_of(gst);
  if (h.mode == BM_DONE || h.mode == BM_CHORD) return;
  const KLayout L = bnd_layout(a, h.pa);
  const int c0 = ba.c0, N4 = L.N4;
  if (c0 >= N4) return;
  const int c1 = min(c0 + W, N4), w = c1 - c0;
  float* K = ba.kw + (long long)bid * ba.kstride;
  float* rinv = carve_state(gst, a).rinv;
  {
    // lane: quad q = lane % 16 of rows r0 + 2·u (u < 32): all loads of a batch in flight first
    const float* Ub = ba.ug + (long long)bid * ba.ustride;
    const int q = tid & 15, rr = tid >> 4;
    const bool qok = 4 * q < w;
#pragma unroll 1
    for (int r0 = rr; r0 < w; r0 += 16 * (NT / 16)) {
      float4 v[16], u[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int r = r0 + t * (NT / 16), i = c0 + r, j = c0 + 4 * q;
        const bool ok = r < w && qok && j <= i;
        v[t] = ok ? *reinterpret_cast<const float4*>(K + L.off(i) + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        u[t] = (ok && c0 > 0) ? *reinterpret_cast<const float4*>(Ub + r * W + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int r = r0 + t * (NT / 16);
        if (r < w)  // the panel's Schur update from bnd_tc_update subtracted
          *reinterpret_cast<float4*>(D + r * DS + 4 * q) =
              make_float4(v[t].x - u[t].x, v[t].y - u[t].y, v[t].z - u[t].z, v[t].w - u[t].w);
      }
    }
  }
  __syncthreads();
  PanelLayout P;
  P.N4 = c1; P.NB = L.NB; P.npos = L.npos; P.c0 = c0; P.S = DS; P.base = L;
  factor_big_range<NT, PanelLayout, QPB200_PDIAG_QS>(D - c0, P, a.floor_rel * h.dmax, rinv, scr, c0, c1);
  __syncthreads();
  for (int b = c0 / KB + (tid >> 5); KB * b < c1; b += NT / 32) invert_diag_block(D - c0, P, b, rinv);
  __syncthreads();
  if (ba.fuse) {
    // the forward substitution of the panel's rows (solve_qd's forward loop
    // on the panel, rows below it in bnd_prows): per 16-block u_b = W_b r_b,
    // then r_i −= L_ib u_b for the panel's rows below the block
    __shared__ float ur[W];
    float* rhs = carve_state(gst, a).rhs;
    for (int e = tid; e < w; e += NT) ur[e] = rhs[c0 + e];
    __syncthreads();
    for (int k0l = 0; k0l < w; k0l += KB) {
      const int kb = min(KB, w - k0l);
      float u = 0.f;
      if (tid < kb) {
        u = rinv[c0 + k0l + tid] * ur[k0l + tid];
        for (int c = 0; c < tid; ++c) u = fmaf(D[(k0l + c) * DS + k0l + tid], ur[k0l + c], u);  // W[t][c], row c col t
      }
      __syncthreads();
      if (tid < kb) ur[k0l + tid] = u;
      __syncthreads();
      for (int il = k0l + KB + tid; il < w; il += NT) {
        float acc = ur[il];
        for (int c = 0; c < kb; ++c) acc = fmaf(-D[il * DS + k0l + c], ur[k0l + c], acc);
        ur[il] = acc;
      }
      __syncthreads();
    }
    for (int e = tid; e < w; e += NT) rhs[c0 + e] = ur[e];
  }
  for (int e = tid; e < w * (W / 4); e += NT) {  // row i keeps columns up to the end of its 16-block
    const int r = e / (W / 4), q = e - r * (W / 4), i = c0 + r, j = c0 + 4 * q;
    if (4 * q < w && j < ((i >> 4) + 1) * KB)
      *reinterpret_cast<float4*>(K + L.off(i) + j) = *reinterpret_cast<const float4*>(D + r * DS + 4 * q);
  }
  if (c1 < N4) {  // rows below follow: the strictly lower part, transposed, for bnd_prows
    float4* dt = reinterpret_cast<float4*>(ba.dtg + (long long)bid * (W * W));
    for (int e = tid; e < W * W / 4; e += NT) {
      const int k = e / (W / 4), j = 4 * (e - k * (W / 4));
      dt[e] = make_float4(k < j ? D[j * DS + k] : 0.f, k < j + 1 ? D[(j + 1) * DS + k] : 0.f,
                          k < j + 2 ? D[(j + 2) * DS + k] : 0.f, k < j + 3 ? D[(j + 3) * DS + k] : 0.f);
    }
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 4) bnd_prows(const BArgs ba) {
  using namespace pnl;
  __shared__ __align__(16) float DT[W * DS];  // DT[k][j] = L[j][k] (j > k): column k contiguous (float4 broadcasts)
  __shared__ float rl[W];
  const Args& a = ba.a;
  const int bid = blockIdx.y, tid = threadIdx.x;
  float* gst = st_of(ba, bid);
  const BScal& h = scal_of(gst);
  if (h.mode == BM_DONE || h.mode == BM_CHORD) return;
  const KLayout L = bnd_layout(a, h.pa);
  const int c0 = ba.c0, N4 = L.N4, c1 = c0 + W;
  const int r0 = c1 + NT * (int)blockIdx.x;
  if (c1 >= N4 || r0 >= N4) return;  // (rows below a panel exist only when it is 64 wide)
  float* K = ba.kw + (long long)bid * ba.kstride;
  const float* rinv = carve_state(gst, a).rinv;
  const float4* dt = reinterpret_cast<const float4*>(ba.dtg + (long long)bid * (W * W));
  {
    static_assert(W * W / 4 % NT == 0 || NT > W * W / 4, "bnd_prows: DT staging");
    constexpr int U = (W * W / 4 + NT - 1) / NT;
    float4 v[U];
#pragma unroll
    for (int t = 0; t < U; ++t) if (tid + t * NT < W * W / 4) v[t] = dt[tid + t * NT];
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const int e = tid + t * NT;
      if (e < W * W / 4) {
        const int k = e / (W / 4), q = e - k * (W / 4);
        *reinterpret_cast<float4*>(DT + k * DS + 4 * q) = v[t];
      }
    }
  }
  for (int k = tid; k < W; k += NT) rl[k] = rinv[c0 + k];
  __shared__ float ur[W];  // the panel's forward-substituted right-hand side (bnd_pdiag, fused)
  float* rhs = carve_state(gst, a).rhs;
  if (ba.fuse)
    for (int k = tid; k < W; k += NT) ur[k] = rhs[c0 + k];
  __syncthreads();
  const int i = r0 + tid;
  if (i >= N4) return;
  float* row = K + L.off(i) + c0;
  float x[W];
  const float4* urow = reinterpret_cast<const float4*>(ba.ug + (long long)bid * ba.ustride + (long long)(i - c0) * W);
#pragma unroll
  for (int q = 0; q < W / 4; ++q) {
    float4 t = reinterpret_cast<const float4*>(row)[q];
    if (c0 > 0) {  // the panel's Schur update from bnd_tc_update
      const float4 u = urow[q];
      t.x -= u.x; t.y -= u.y; t.z -= u.z; t.w -= u.w;
    }
    x[4 * q] = t.x; x[4 * q + 1] = t.y; x[4 * q + 2] = t.z; x[4 * q + 3] = t.w;
  }
#pragma unroll
  for (int k = 0; k < W; ++k) {
    x[k] *= rl[k];
    const float xk = -x[k];
#pragma unroll
    for (int j4 = (k + 1) >> 2; j4 < W / 4; ++j4) {
      const float4 d = *reinterpret_cast<const float4*>(DT + k * DS + 4 * j4);
      if (4 * j4 > k) x[4 * j4] = fmaf(xk, d.x, x[4 * j4]);
      if (4 * j4 + 1 > k) x[4 * j4 + 1] = fmaf(xk, d.y, x[4 * j4 + 1]);
      if (4 * j4 + 2 > k) x[4 * j4 + 2] = fmaf(xk, d.z, x[4 * j4 + 2]);
      x[4 * j4 + 3] = fmaf(xk, d.w, x[4 * j4 + 3]);
    }
  }
  float ri = ba.fuse ? rhs[i] : 0.f;
#pragma unroll
  for (int q = 0; q < W / 4; ++q) {
    const float s0 = sgn_of(c0 + 4 * q, L.npos);  // S_k (npos is a multiple of 4)
    const float4 l = make_float4(s0 * x[4 * q], s0 * x[4 * q + 1], s0 * x[4 * q + 2], s0 * x[4 * q + 3]);
    reinterpret_cast<float4*>(row)[q] = l;
    if (ba.fuse) {  // r_i −= L_i,panel u_panel (fused forward substitution)
      ri = fmaf(-l.x, ur[4 * q], ri); ri = fmaf(-l.y, ur[4 * q + 1], ri);
      ri = fmaf(-l.z, ur[4 * q + 2], ri); ri = fmaf(-l.w, ur[4 * q + 3], ri);
    }
  }
  if (ba.fuse) rhs[i] = ri;
}

// ---------------------------------------------------------------------------
// bnd_sgemm: C[M×N] = A[M×K] · op(B) in FP32 (FMA, the arithmetic of the
// per-problem GEMVs it replaces), op(B) = Bᵀ for B [N×K] (BT) or B [K×N].
// With Q and G shared by the batch (config 4) the residual products of all
// problems are GEMMs: G X, Q X (NT) and Gᵀ Z, Gᵀ T (NN) with the problems'
// x, z, t rows read in place from their state blocks (lda = state stride):
// the shared matrix is read once per 64-problem tile instead of once per
// problem.  64×64 tiles, K in steps of 16, 256 threads with 4×4 outputs each
// (float4 operand reads from shared memory, float4 stores).
// ---------------------------------------------------------------------------
template <bool BT>
__global__ void __launch_bounds__(256) bnd_sgemm(const float* __restrict__ A, long long lda,
                                                 const float* __restrict__ B, long long ldb, float* __restrict__ C,
                                                 long long ldc, int M, int N, int K) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ __align__(16) float As[BK][BM + 4], Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const bool va = !(lda & 3) && !(reinterpret_cast<uintptr_t>(A) & 15);
  const bool vb = !(ldb & 3) && !(reinterpret_cast<uintptr_t>(B) & 15);
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    {  // A tile: row r = tid / 4, k quad (tid % 4)·4, stored k-major
      const int r = tid >> 2, kq = (tid & 3) * 4, gm = m0 + r, gk = k0 + kq;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gm < M) {
        const float* src = A + (long long)gm * lda + gk;
        if (va && gk + 3 < K) v = *reinterpret_cast<const float4*>(src);
        else {
          if (gk < K) v.x = src[0];
          if (gk + 1 < K) v.y = src[1];
          if (gk + 2 < K) v.z = src[2];
          if (gk + 3 < K) v.w = src[3];
        }
      }
      As[kq][r] = v.x; As[kq + 1][r] = v.y; As[kq + 2][r] = v.z; As[kq + 3][r] = v.w;
    }
    if constexpr (BT) {  // B [N×K]: like A
      const int r = tid >> 2, kq = (tid & 3) * 4, gn = n0 + r, gk = k0 + kq;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gn < N) {
        const float* src = B + (long long)gn * ldb + gk;
        if (vb && gk + 3 < K) v = __ldg(reinterpret_cast<const float4*>(src));
        else {
          if (gk < K) v.x = __ldg(src);
          if (gk + 1 < K) v.y = __ldg(src + 1);
          if (gk + 2 < K) v.z = __ldg(src + 2);
          if (gk + 3 < K) v.w = __ldg(src + 3);
        }
      }
      Bs[kq][r] = v.x; Bs[kq + 1][r] = v.y; Bs[kq + 2][r] = v.z; Bs[kq + 3][r] = v.w;
    } else {  // B [K×N]: k row tid / 16, column quad (tid % 16)·4
      const int kr = tid >> 4, nq = (tid & 15) * 4, gk = k0 + kr, gn = n0 + nq;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < K) {
        const float* src = B + (long long)gk * ldb + gn;
        if (vb && gn + 3 < N) v = __ldg(reinterpret_cast<const float4*>(src));
        else {
          if (gn < N) v.x = __ldg(src);
          if (gn + 1 < N) v.y = __ldg(src + 1);
          if (gn + 2 < N) v.z = __ldg(src + 2);
          if (gn + 3 < N) v.w = __ldg(src + 3);
        }
      }
      *reinterpret_cast<float4*>(&Bs[kr][nq]) = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {  // thread (ty, tx): rows 4·ty + [0, 4), columns 4·tx + [0, 4)
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][4 * ty]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][4 * tx]);
      const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  const bool vc = !(ldc & 3) && !(reinterpret_cast<uintptr_t>(C) & 15);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + 4 * ty + i, gn = n0 + 4 * tx;
    if (gm >= M) continue;
    float* dst = C + (long long)gm * ldc + gn;
    if (vc && gn + 3 < N) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (gn + j < N) dst[j] = acc[i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// bnd_cache: grid (chunks, B), after the panel loop of a solve iteration in
// which some problems reached κ < √10·κ_relax for the first time (reading
// Q26): their factor (packed L), pivot reciprocals, partition and Jacobian
// vectors go to the chord cache that the backward's chord steps solve with.
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT) bnd_cache(const BArgs ba) {
  const Args& a = ba.a;
  const int bid = blockIdx.y, tid = threadIdx.x;
  float* gst = st_of(ba, bid);
  const BScal& h = scal_of(gst);
  if (h.mode != BM_NEWTON || !h.cache_now) return;
  const KLayout L = bnd_layout(a, h.pa);
  const float4* src = reinterpret_cast<const float4*>(ba.kw + (long long)bid * ba.kstride);
  float4* dst = reinterpret_cast<float4*>(a.kc + (long long)bid * a.kc_stride);
  const int n4v = (L.size() + 3) >> 2;
  for (int i = blockIdx.x * NT + tid; i < n4v; i += gridDim.x * NT) dst[i] = src[i];
  if (blockIdx.x == 0) {
    const Smem S = carve_state(gst, a);
    float* cj = a.chd + (long long)bid * a.chd_stride;
    const int p = a.p, p4 = (p + 3) & ~3;
    for (int i = tid; i < p; i += NT) {
      cj[4 + i] = S.dp[i]; cj[4 + p4 + i] = S.dm[i]; cj[4 + 2 * p4 + i] = S.c[i];
      cj[4 + 3 * p4 + i] = __int_as_float(S.widx[i]);
    }
    for (int i = tid; i < L.N4; i += NT) cj[4 + 4 * p4 + i] = S.rinv[i];
    if (tid == 0) {
      cj[0] = __int_as_float(h.pa); cj[1] = h.kappa;
      a.chord_ok[bid] = 1;
    }
  }
}

// ---------------------------------------------------------------------------
// bnd_solve: grid B — forward and backward substitution with the factor
// (solve_qd), right-hand side staged in shared memory.
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT) bnd_solve(const BArgs ba) {
  extern __shared__ __align__(16) float sm[];
  const Args& a = ba.a;
  const int bid = blockIdx.x;
  float* gst = st_of(ba, bid);
  const BScal& h = scal_of(gst);
  if (h.mode == BM_DONE) return;
  const KLayout L = bnd_layout(a, h.pa);
  const Smem G = carve_state(gst, a);
  const bool chord = h.mode == BM_CHORD;  // the cached factorisation of the solve (reading Q26)
  const float* K = chord ? a.kc + (long long)bid * a.kc_stride : ba.kw + (long long)bid * ba.kstride;
  const float* rinv = chord ? a.chd + (long long)bid * a.chd_stride + 4 + 4 * ((a.p + 3) & ~3) : G.rinv;
  copy_block<NT>(sm, G.rhs, L.N4);
  if (ba.pre && chord) {  // + Gᵀ t of the batched GEMM (residuals, pre; bnd_scatter adds it for a Newton step)
    const float* gt = ba.pre + (long long)bid * ba.pre_stride + 2 * a.n4;
    for (int j = threadIdx.x; j < a.n; j += NT) sm[j] += gt[j];
    __syncthreads();
  }
  solve_qd<NT, false, true>(K, L, rinv, sm, nullptr, !(ba.fuse && !chord));
  __syncthreads();
  copy_block<NT>(G.rhs, sm, L.N4);
}

// ---------------------------------------------------------------------------
// bnd_update: grid B — the tail of the loop body: the initial point (INIT),
// the Newton step with its fraction-to-boundary step length and retraction
// (NEWTON), or Alg. 3's gradients from the relaxed factorisation (ADJ).
// ---------------------------------------------------------------------------
template <int NT, bool LARGE = false>
__global__ void __launch_bounds__(NT) bnd_update(const BArgs ba) {
  extern __shared__ __align__(16) float sm[];
  const Args& a = ba.a;
  const int bid = blockIdx.x, tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, m = a.m, p = a.p;
  float* gst = st_of(ba, bid);
  if (scal_of(gst).mode == BM_DONE) return;
  copy_block<NT>(sm, gst, ba.st_stride);
  const Smem S = carve_state(sm, a);
  BScal& h = scal_of(sm);
  const Prob P = prob_of(a, bid);
  const bool bwd = a.bwd != 0;
  const int mode = h.mode, pa = h.pa;
  if (mode == BM_INIT) {
    for (int j = tid; j < n; j += NT) S.x[j] = S.rhs[j];
    for (int l = tid; l < m; l += NT) S.y[l] = S.rhs[n4 + l];
    __syncthreads();
    if (ba.pre) {  // G x from the batched GEMM after bnd_solve (x = the solve's rhs)
      for (int i = tid; i < p; i += NT) S.dz[i] = S.gx[i];
      __syncthreads();
    } else {
      if constexpr (LARGE) rowdots_large<NT>(P.G, p, n, S.x, S.dz);
      else rowdots<NT>(P.G, p, n, S.x, S.dz);
    }
    for (int i = tid; i < p; i += NT) S.dz[i] -= __ldg(P.h + i);  // ẑ = Gx − h
    __syncthreads();
    float ap = -INFINITY, ad = -INFINITY, bad = 0.f;
    for (int i = tid; i < p; i += NT) {
      const float zh = S.dz[i];
      ap = fmaxf(ap, zh); ad = fmaxf(ad, -zh);
      if (!isfinite(zh)) bad = 1.f;
    }
    for (int j = tid; j < n; j += NT) if (!isfinite(S.x[j])) bad = 1.f;
    float v[3] = {ap, ad, bad};
    block_reduce<NT, 0, 3>(v, S.red);
    for (int i = tid; i < p; i += NT) {  // s~ = −ẑ, z~ = ẑ, shifted into the interior
      const float zh = S.dz[i];
      S.s[i] = v[0] >= 0.f ? -zh + (1.f + v[0]) : -zh;
      S.z[i] = v[1] >= 0.f ? zh + (1.f + v[1]) : zh;
    }
    __syncthreads();
    if (v[2] > 0.f) {
      if (tid == 0) { h.status = ST_FAIL | (STG_INIT << 8); h.it = 0; }
      __syncthreads();
      bnd_finish_solve<NT>(a, S, h, bid);
    } else if (tid == 0) {
      h.mode = BM_NEWTON;
    }
  } else if (mode == BM_NEWTON || mode == BM_CHORD) {
    float kappa = h.kappa;
    int stage = 0;
    const bool okstep = newton_update<NT, LARGE>(S, a, P, pa, kappa, kappa - h.kt, &stage, ba.pre != nullptr);
    if (!okstep) {
      if (tid == 0) h.status = ST_FAIL | ((bwd ? STG_RELAX : stage) << 8);
      __syncthreads();
      if (!bwd) bnd_finish_solve<NT>(a, S, h, bid);
      else bnd_finish_backward<NT>(a, S, h, bid);
    } else if (tid == 0) {
      h.kappa = kappa;
    }
  } else {  // BM_ADJ: dv = G dx + w (f2 = 0), dz = d₊ ⊙ dv (reading Q8), Alg. 3 outer products
    recover_dv<NT, LARGE>(S, a, P, true, ba.pre != nullptr);
    for (int i = tid; i < p; i += NT) S.dz[i] = S.dp[i] * S.gx[i];
    for (int j = tid; j < n; j += NT) S.dx[j] = S.rhs[j];
    for (int l = tid; l < m; l += NT) S.dy[l] = S.rhs[n4 + pa + l];
    __syncthreads();
    float bad = 0.f;
    for (int j = tid; j < n; j += NT) if (!isfinite(S.dx[j])) bad = 1.f;
    for (int i = tid; i < p; i += NT) if (!isfinite(S.dz[i])) bad = 1.f;
    for (int l = tid; l < m; l += NT) if (!isfinite(S.dy[l])) bad = 1.f;
    float v[1] = {bad};
    block_reduce<NT, 0, 1>(v, S.red);
    if (tid == 0) {
      h.ok = !(v[0] > 0.f);
      if (!h.ok) h.status = ST_FAIL | (STG_BACKWARD << 8);
    }
    __syncthreads();
    bnd_finish_backward<NT>(a, S, h, bid);
  }
  __syncthreads();
  copy_block<NT>(gst, sm, ba.st_stride);
}

}  // namespace qpb

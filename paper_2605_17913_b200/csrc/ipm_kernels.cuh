// ipm_kernels.cuh — the persistent per-problem IPM kernels (solve: init +
// Alg. 1; backward: Alg. 2 + Alg. 3) and the batch-sum kernel for gradients
// of shared parameters.  One CTA owns one QP for the whole kernel; the KKT
// matrix, the iterate and all per-iteration vectors live in shared memory;
// the problem data (Q, G, A, …) is re-read from global memory (L2) each
// iteration.  See DESIGN.md §5 for the data layout and §6 for the roofline.
#pragma once
#include "ipm_cta.cuh"

namespace qpb {

enum { ST_CONVERGED = 0, ST_MAX_ITER = 2, ST_FAIL = 3 };
enum { STG_SCALING = 1, STG_PREDICTOR = 2, STG_CENTERING = 3, STG_CORRECTOR = 4, STG_LINESEARCH = 5,
       STG_RELAX = 6, STG_BACKWARD = 7, STG_INIT = 8 };

struct Args {
  int B, n, m, p;
  int n4, nw, N, N4;      // KKT layout (nw = p for the implicit form)
  KLayout kl;             // packed block layout of the KKT lower triangle
  const float *Q, *q, *A, *b, *G, *h;
  long long sQ, sq, sA, sb, sG, sh;
  float *x, *y, *z, *s;  // solution (solve: out; backward: in)
  int *iters, *status;
  const float* dl;
  float *gQ, *gq, *gA, *gb, *gG, *gh;        // per-problem gradients (nullptr = skip)
  float *wx, *wy, *wz, *wdx, *wdy, *wdz;     // per-problem vectors for shared sums (nullptr = skip)
  int *riters, *rstatus;
  float tol, sigma, tau, kappa_relax, relax_ktol, floor_rel, relax_tol;
  int max_iter, relax_max_iter;
};

// Shared-memory carve-up (floats).  Every segment is a multiple of 4 floats
// so that float4 accesses stay 16-byte aligned.  layout() is used by the host
// (base = nullptr, to size the allocation) and by the kernels.
struct Smem {
  float *K, *rinv, *rhs;
  float *x, *y, *z, *s, *v, *dp, *dm, *c;
  float *rt, *re, *ri, *rz, *rs;
  float *dx, *dy, *dz, *ds, *dv, *t, *mx;
  float* red;
  int* flag;
  float* end;
};

__host__ __device__ inline Smem layout(float* base, int n4, int m, int p, int N4, int ksize) {
  const int m4 = (m + 3) & ~3, p4 = (p + 3) & ~3;
  Smem S;
  float* q = base;
  S.K = q; q += ksize;
  S.rinv = q; q += N4;
  S.rhs = q; q += N4;
  S.x = q; q += n4;
  S.y = q; q += m4;
  S.z = q; q += p4;
  S.s = q; q += p4;
  S.v = q; q += p4;
  S.dp = q; q += p4;
  S.dm = q; q += p4;
  S.c = q; q += p4;
  S.rt = q; q += n4;
  S.re = q; q += m4;
  S.ri = q; q += p4;
  S.rz = q; q += p4;
  S.rs = q; q += p4;
  S.dx = q; q += n4;
  S.dy = q; q += m4;
  S.dz = q; q += p4;
  S.ds = q; q += p4;
  S.dv = q; q += p4;
  S.t = q; q += p4;
  S.mx = q; q += p4 + m4;
  S.red = q; q += 160;
  S.flag = reinterpret_cast<int*>(q); q += 4;
  S.end = q;
  return S;
}

__host__ inline size_t ipm_smem_bytes(int n4, int m, int p, int N4, int ksize) {
  const Smem S = layout(nullptr, n4, m, p, N4, ksize);
  return (size_t)(reinterpret_cast<uintptr_t>(S.end)) ;
}

__device__ inline Smem carve(float* base, const Args& a) { return layout(base, a.n4, a.m, a.p, a.N4, a.kl.size()); }

struct Prob {
  const float *Q, *q, *A, *b, *G, *h;
};

__device__ __forceinline__ Prob prob_of(const Args& a, int bid) {
  Prob P;
  P.Q = a.Q + a.sQ * bid; P.q = a.q + a.sq * bid; P.A = a.A + a.sA * bid;
  P.b = a.b + a.sb * bid; P.G = a.G + a.sG * bid; P.h = a.h + a.sh * bid;
  return P;
}

// ------------------------------------------------------------------------
// KKT assembly (bounded scaling): the lower triangle of
//   [[Q + Gᵀ diag(wH) G, Gᵀ diag(wC), Aᵀ], [diag(wC) G, −diag(e), 0], [A, 0, 0]]
// Implicit Newton step: wH = wC = d₊, e = d₋ (the M form).  CVXOPT init
// (congruent form of [[Q,Gᵀ,Aᵀ],[G,−I,0],[A,0,0]]): wH = 1, wC = 0, e = 1.
// Returns max|diag| over the real rows (for the pivot floor).
// ------------------------------------------------------------------------
template <int NT>
__device__ float assemble(const Smem& S, const Args& a, const Prob& P, const float* wH, const float* wC,
                          const float* e, bool unit_wH, bool zero_wC) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.nw, m = a.m, N = a.N, N4 = a.N4;
  const KLayout& L = a.kl;
  float* K = S.K;
  // 1. stage raw G into the C block rows [n4, n4+p), cols [0, n4) (zero pad)
  for (int idx = tid; idx < p * n4; idx += NT) {
    const int k = idx / n4, j = idx - k * n4;
    K[L.off(n4 + k) + j] = j < n ? __ldg(P.G + k * n + j) : 0.f;
  }
  // rows ≥ n4: A rows, zeros / −e on the w,y blocks, −1 on padding rows;
  // every row's tail beyond the diagonal (rest of its diagonal block + pad) is zeroed
  for (int r = n4 + tid; r < N4; r += NT) {
    float* row = K + L.off(r);
    const int len = L.len(r >> 4);
    if (r >= n4 + p && r < N) {
      const int l = r - n4 - p;
      for (int j = 0; j < n4; ++j) row[j] = j < n ? __ldg(P.A + l * n + j) : 0.f;
    }
    if (r >= N) for (int j = 0; j < n4; ++j) row[j] = 0.f;
    for (int j = n4; j < len; ++j) row[j] = 0.f;
    if (r < n4 + p) row[r] = -e[r - n4];
    else if (r >= N) row[r] = -1.f;
  }
  __syncthreads();
  // 2. H = Q + Gᵀ diag(wH) G, aligned 4×4 tiles of the lower triangle (x-block rows
  //    also get their tails beyond the diagonal zeroed)
  const int T = n4 >> 2;
  const int nt = T * (T + 1) / 2;
  float dmax = 0.f;
  for (int t = tid; t < nt; t += NT) {
    int I = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;
    const int i0 = 4 * I, j0 = 4 * J;
    float acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int i = i0 + u, j = j0 + w;
        acc[u][w] = (i < n && j < n) ? __ldg(P.Q + i * n + j) : (i == j ? 1.f : 0.f);
      }
    for (int k = 0; k < p; ++k) {
      const float* gk = K + L.off(n4 + k);
      const float4 gi = *reinterpret_cast<const float4*>(gk + i0);
      float4 gj = *reinterpret_cast<const float4*>(gk + j0);
      if (!unit_wH) {
        const float w = wH[k];
        gj.x *= w; gj.y *= w; gj.z *= w; gj.w *= w;
      }
      const float gia[4] = {gi.x, gi.y, gi.z, gi.w};
      const float gja[4] = {gj.x, gj.y, gj.z, gj.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] = fmaf(gia[u], gja[w], acc[u][w]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float* row = K + L.off(i0 + u);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int i = i0 + u, j = j0 + w;
        if (j <= i) row[j] = acc[u][w];
        if (i == j && i < n) dmax = fmaxf(dmax, fabsf(acc[u][w]));
      }
      if (I == J) {  // zero the tail of row i0+u beyond the diagonal
        const int len = L.len((i0 + u) >> 4);
        for (int j = i0 + u + 1; j < len; ++j) row[j] = 0.f;
      }
    }
  }
  __syncthreads();
  // 3. C block scaled in place: diag(wC) G
  for (int idx = tid; idx < p * n4; idx += NT) {
    const int k = idx / n4, j = idx - k * n4;
    float* el = K + L.off(n4 + k) + j;
    *el = zero_wC ? 0.f : *el * wC[k];
  }
  for (int k = tid; k < p; k += NT) dmax = fmaxf(dmax, fabsf(e[k]));
  float vals[1] = {dmax};
  block_reduce<NT, 0, 1>(vals, S.red);
  return vals[0];
}

// Warp-per-row dot products out[r] = Mat[r,:]·vec for r < rows (Mat global,
// row-major rows×n, vec in smem); fn(r, dot) runs on lane 0.
template <int NT, typename F>
__device__ __forceinline__ void rowdots(const float* __restrict__ Mat, int rows, int n, const float* vec, F fn) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < rows; r += NT / 32) {
    const float* row = Mat + r * n;
    float acc = 0.f;
    for (int j = lane; j < n; j += 32) acc = fmaf(__ldg(row + j), vec[j], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) fn(r, acc);
  }
}

// ------------------------------------------------------------------------
// Residuals (Eq. 4; Eq. 10), the relative stopping test
// (reading Q4) and the Newton right-hand side of Eq. 14 in the
// M coordinates: rhs = (−(r_t − Gᵀ(r_z + c r_κ)), −(r_i − r_s − c r_κ), −r_e).
// Also fills d₊, d₋, c at (v, κ).  Returns the norms (block-uniform).
// ------------------------------------------------------------------------
struct Norms {
  float gap, obj, nonfin;
  float nrt, nre, nri, nrzs, sQx, sq, sGz, sAy, sAx, sb, sGx, ss, sh, sz;
};

template <int NT>
__device__ Norms residuals(const Smem& S, const Args& a, const Prob& P, float kappa, float r_kappa) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  float mz = 0.f, ms = 0.f, mh = 0.f, mrzs = 0.f, nonfin = 0.f;
  // elementwise: r_z, r_s, d±, c, t = r_z + c r_κ
  for (int k = tid; k < p; k += NT) {
    const float zk = S.z[k], sk = S.s[k], vk = S.v[k];
    const float rz = zk - ret_b(vk, kappa), rs = sk - ret_b(-vk, kappa);
    const float c = ret_dk(vk, kappa);
    S.rz[k] = rz; S.rs[k] = rs; S.c[k] = c;
    S.dp[k] = ret_db(vk, kappa); S.dm[k] = ret_db(-vk, kappa);
    S.t[k] = fmaf(c, r_kappa, rz);
    mz = fmaxf(mz, fabsf(zk)); ms = fmaxf(ms, fabsf(sk)); mh = fmaxf(mh, fabsf(__ldg(P.h + k)));
    mrzs = fmaxf(mrzs, fmaxf(fabsf(rz), fabsf(rs)));
  }
  __syncthreads();
  // columns j < n: Qx, Gᵀz, Aᵀy, Gᵀt  (Q symmetric ⇒ (Qx)_j = Σ_i Q_ij x_i)
  float mrt = 0.f, mqx = 0.f, mq = 0.f, mgz = 0.f, may = 0.f, obj = 0.f;
  for (int j = tid; j < n; j += NT) {
    float qx = 0.f, gz = 0.f, gt = 0.f, ay = 0.f;
    for (int i = 0; i < n; ++i) qx = fmaf(__ldg(P.Q + i * n + j), S.x[i], qx);
    for (int k = 0; k < p; ++k) {
      const float g = __ldg(P.G + k * n + j);
      gz = fmaf(g, S.z[k], gz);
      gt = fmaf(g, S.t[k], gt);
    }
    for (int l = 0; l < m; ++l) ay = fmaf(__ldg(P.A + l * n + j), S.y[l], ay);
    const float qj = __ldg(P.q + j);
    const float rt = qx + qj + gz + ay;
    S.rt[j] = rt;
    S.rhs[j] = -(rt - gt);
    mrt = fmaxf(mrt, fabsf(rt)); mqx = fmaxf(mqx, fabsf(qx)); mq = fmaxf(mq, fabsf(qj));
    mgz = fmaxf(mgz, fabsf(gz)); may = fmaxf(may, fabsf(ay));
    obj = fmaf(S.x[j], fmaf(0.5f, qx, qj), obj);
    if (!isfinite(rt)) nonfin += 1.f;
  }
  for (int j = n + tid; j < n4; j += NT) S.rhs[j] = 0.f;
  for (int j = a.N + tid; j < a.N4; j += NT) S.rhs[j] = 0.f;
  // rows: r_i = Gx + s − h, r_e = Ax − b  (warp per row)
  float* mx = S.mx;  // per-row |Gx| / |Ax| stash
  rowdots<NT>(P.G, p, n, S.x, [&](int k, float gx) {
    const float ri = gx + S.s[k] - __ldg(P.h + k);
    S.ri[k] = ri;
    S.rhs[n4 + k] = -(ri - S.rs[k] - S.c[k] * r_kappa);
    mx[k] = gx;
  });
  rowdots<NT>(P.A, m, n, S.x, [&](int l, float ax) {
    const float re = ax - __ldg(P.b + l);
    S.re[l] = re;
    S.rhs[n4 + p + l] = -re;
    mx[p + l] = ax;
  });
  __syncthreads();
  float mri = 0.f, mgx = 0.f, mre = 0.f, max_ = 0.f, mb = 0.f, gap = 0.f;
  for (int k = tid; k < p; k += NT) {
    mri = fmaxf(mri, fabsf(S.ri[k])); mgx = fmaxf(mgx, fabsf(mx[k]));
    gap = fmaf(S.s[k], S.z[k], gap);
  }
  for (int l = tid; l < m; l += NT) {
    mre = fmaxf(mre, fabsf(S.re[l])); max_ = fmaxf(max_, fabsf(mx[p + l])); mb = fmaxf(mb, fabsf(__ldg(P.b + l)));
  }
  float v[17] = {gap, obj, nonfin, mrt, mre, mri, mrzs, mqx, mq, mgz, may, max_, mb, mgx, ms, mh, mz};
  block_reduce<NT, 3, 14>(v, S.red);
  Norms R;
  R.gap = v[0]; R.obj = v[1]; R.nonfin = v[2]; R.nrt = v[3]; R.nre = v[4]; R.nri = v[5]; R.nrzs = v[6];
  R.sQx = v[7]; R.sq = v[8]; R.sGz = v[9]; R.sAy = v[10]; R.sAx = v[11]; R.sb = v[12]; R.sGx = v[13];
  R.ss = v[14]; R.sh = v[15]; R.sz = v[16];
  return R;
}

__device__ __forceinline__ bool feasible_rel(const Norms& R, float tol) {
  const float st = fmaxf(1.f, fmaxf(fmaxf(R.sQx, R.sq), fmaxf(R.sGz, R.sAy)));
  const float se = fmaxf(1.f, fmaxf(R.sAx, R.sb));
  const float si = fmaxf(1.f, fmaxf(R.sGx, fmaxf(R.ss, R.sh)));
  const float sz = fmaxf(1.f, fmaxf(R.sz, R.ss));
  return R.nrt <= tol * st && R.nre <= tol * se && R.nri <= tol * si && R.nrzs <= tol * sz;
}
// phi = largest of the four relative residuals (feasible_rel <=> phi <= tol).
__device__ __forceinline__ float rel_phi(const Norms& R) {
  const float st = fmaxf(1.f, fmaxf(fmaxf(R.sQx, R.sq), fmaxf(R.sGz, R.sAy)));
  const float se = fmaxf(1.f, fmaxf(R.sAx, R.sb));
  const float si = fmaxf(1.f, fmaxf(R.sGx, fmaxf(R.ss, R.sh)));
  const float sz = fmaxf(1.f, fmaxf(R.sz, R.ss));
  return fmaxf(fmaxf(R.nrt / st, R.nre / se), fmaxf(R.nri / si, R.nrzs / sz));
}
// Reading Q5b: Alg. 2 stops (with κ at κ_relax) when phi <= relax_tol, or
// phi <= tol and the last Newton step did not reduce phi by 10% (f32 floor).
__device__ __forceinline__ bool relax_done(const Norms& R, float tol, float relax_tol, float phi_prev) {
  const float phi = rel_phi(R);
  return phi <= relax_tol || (phi <= tol && phi > 0.9f * phi_prev);
}
__device__ __forceinline__ bool converged_solve(const Norms& R, float tol) {
  return feasible_rel(R, tol) && R.gap <= tol * fmaxf(1.f, fabsf(R.obj));
}

// v = z − s and κ = sᵀz/p (Alg. 1 lines 5-6; divisor p: reading Q1)
template <int NT>
__device__ float manifold_coords(const Smem& S, const Args& a) {
  float gap = 0.f;
  for (int k = threadIdx.x; k < a.p; k += NT) {
    S.v[k] = S.z[k] - S.s[k];
    gap = fmaf(S.s[k], S.z[k], gap);
  }
  float v[1] = {gap};
  block_reduce<NT, 1, 0>(v, S.red);
  return a.p > 0 ? v[0] / (float)a.p : 0.f;
}

// After solve_qd: Δx = rhs[0:n], w = rhs[n4:n4+p], Δy = rhs[n4+p:N];
// Δv = GΔx + w; Δκ = −r_κ; Δz = −r_z + d₊Δv + cΔκ; Δs = −r_s − d₋Δv + cΔκ
// (Eq. 13 rows 4-6).  Then α = min(1, τ α_max) (Eq. 6 + Q3), the step on
// (x, y, v, κ) and the retraction.  Returns false (and leaves the
// iterate untouched) if the direction is not finite.
template <int NT>
__device__ bool newton_update(const Smem& S, const Args& a, const Prob& P, float& kappa, float r_kappa,
                              int* stage) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  const float dk = -r_kappa;
  rowdots<NT>(P.G, p, n, S.rhs, [&](int k, float gdx) { S.dv[k] = gdx + S.rhs[n4 + k]; });
  __syncthreads();
  float amax = INFINITY, bad = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float dv = S.dv[k];
    const float dz = -S.rz[k] + S.dp[k] * dv + S.c[k] * dk;
    const float ds = -S.rs[k] - S.dm[k] * dv + S.c[k] * dk;
    S.dz[k] = dz; S.ds[k] = ds;
    if (ds < 0.f) amax = fminf(amax, -S.s[k] / ds);
    if (dz < 0.f) amax = fminf(amax, -S.z[k] / dz);
    if (!isfinite(dz) || !isfinite(ds)) bad = 1.f;
  }
  for (int j = tid; j < n; j += NT) if (!isfinite(S.rhs[j])) bad = 1.f;
  for (int l = tid; l < m; l += NT) if (!isfinite(S.rhs[n4 + p + l])) bad = 1.f;
  float vals[1] = {bad};
  block_reduce<NT, 0, 1>(vals, S.red);
  const float am = block_min<NT>(amax, S.red + 64);
  if (vals[0] > 0.f) { *stage = STG_CORRECTOR; return false; }
  const float alpha = fminf(1.f, a.tau * am);
  if (!(alpha > 0.f)) { *stage = STG_LINESEARCH; return false; }
  for (int j = tid; j < n; j += NT) S.x[j] = fmaf(alpha, S.rhs[j], S.x[j]);
  for (int l = tid; l < m; l += NT) S.y[l] = fmaf(alpha, S.rhs[n4 + p + l], S.y[l]);
  const float kn = fmaf(alpha, dk, kappa);
  for (int k = tid; k < p; k += NT) {
    const float vn = fmaf(alpha, S.dv[k], S.v[k]);
    S.z[k] = ret_b(vn, kn);
    S.s[k] = ret_b(-vn, kn);
  }
  kappa = kn;
  __syncthreads();
  return true;
}

// ------------------------------------------------------------------------
// Kernel: initialisation (Q11) + Algorithm 1.
// ------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT, 3) ipm_solve_kernel(const Args a) {
  extern __shared__ __align__(16) float smem[];
  const int bid = blockIdx.x;
  const int tid = threadIdx.x;
  const Smem S = carve(smem, a);
  const Prob P = prob_of(a, bid);
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  int status = ST_CONVERGED, it = 0;

  // ---- initialisation: solve [[Q, Gᵀ, Aᵀ], [G, −I, 0], [A, 0, 0]] (x, ẑ, y) = (−q, h, b)
  // in the congruent form M(wH=1, wC=0, e=1)(x, w, y) = (−q + Gᵀh, h, b), ẑ = Gx + w = Gx − h.
  for (int k = tid; k < p; k += NT) S.t[k] = 1.f;
  __syncthreads();
  {
    const float dmax = assemble<NT>(S, a, P, S.t, S.t, S.t, true, true);
    for (int j = tid; j < n4; j += NT) {
      float acc = 0.f;
      if (j < n) {
        acc = -__ldg(P.q + j);
        for (int k = 0; k < p; ++k) acc = fmaf(__ldg(P.G + k * n + j), __ldg(P.h + k), acc);
      }
      S.rhs[j] = acc;
    }
    for (int k = tid; k < p; k += NT) S.rhs[n4 + k] = __ldg(P.h + k);
    for (int l = tid; l < m; l += NT) S.rhs[n4 + p + l] = __ldg(P.b + l);
    for (int j = a.N + tid; j < a.N4; j += NT) S.rhs[j] = 0.f;
    factor_qd<NT>(S.K, a.kl, a.floor_rel * dmax, S.rinv, S.flag);
    solve_qd<NT>(S.K, a.kl, S.rinv, S.rhs);
    for (int j = tid; j < n; j += NT) S.x[j] = S.rhs[j];
    for (int l = tid; l < m; l += NT) S.y[l] = S.rhs[n4 + p + l];
    __syncthreads();
    rowdots<NT>(P.G, p, n, S.x, [&](int k, float gx) { S.dz[k] = gx - __ldg(P.h + k); });  // ẑ
    __syncthreads();
    float ap = -INFINITY, ad = -INFINITY, bad = 0.f;
    for (int k = tid; k < p; k += NT) {
      const float zh = S.dz[k];
      ap = fmaxf(ap, zh); ad = fmaxf(ad, -zh);
      if (!isfinite(zh)) bad = 1.f;
    }
    for (int j = tid; j < n; j += NT) if (!isfinite(S.x[j])) bad = 1.f;
    float v[3] = {ap, ad, bad};
    block_reduce<NT, 0, 3>(v, S.red);
    ap = v[0]; ad = v[1];
    for (int k = tid; k < p; k += NT) {
      const float zh = S.dz[k];
      S.s[k] = ap >= 0.f ? -zh + (1.f + ap) : -zh;
      S.z[k] = ad >= 0.f ? zh + (1.f + ad) : zh;
    }
    __syncthreads();
    if (v[2] > 0.f) status = ST_FAIL | (STG_INIT << 8);
  }

  // ---- Algorithm 1 -----------------------------------------------------------
  if (status == ST_CONVERGED) {
    for (int k = 0;; ++k) {
      float kappa = manifold_coords<NT>(S, a);
      const float kt = a.sigma * kappa;  // κ_target = σκ
      const Norms R = residuals<NT>(S, a, P, kappa, kappa - kt);
      it = k;
      if (R.nonfin > 0.f) { status = ST_FAIL | (STG_SCALING << 8); break; }
      if (converged_solve(R, a.tol)) { status = ST_CONVERGED; break; }
      if (k == a.max_iter) { status = ST_MAX_ITER; break; }
      const float dmax = assemble<NT>(S, a, P, S.dp, S.dp, S.dm, false, false);
      factor_qd<NT>(S.K, a.kl, a.floor_rel * dmax, S.rinv, S.flag);
      solve_qd<NT>(S.K, a.kl, S.rinv, S.rhs);
      int stage = 0;
      if (!newton_update<NT>(S, a, P, kappa, kappa - kt, &stage)) { status = ST_FAIL | (stage << 8); break; }
    }
  }
  // ---- outputs
  for (int j = tid; j < n; j += NT) a.x[(long long)bid * n + j] = S.x[j];
  for (int l = tid; l < m; l += NT) a.y[(long long)bid * m + l] = S.y[l];
  for (int k = tid; k < p; k += NT) {
    a.z[(long long)bid * p + k] = S.z[k];
    a.s[(long long)bid * p + k] = S.s[k];
  }
  if (tid == 0) {
    a.iters[bid] = it;
    a.status[bid] = status;
  }
}

// ------------------------------------------------------------------------
// Kernel: Algorithm 2 (relax, exact Newton, factor-then-check: Q5, Q6) and
// Algorithm 3 (sign reading Q7, dz = d₊⊙dv: Q8).
// ------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(NT, 3) ipm_backward_kernel(const Args a) {
  extern __shared__ __align__(16) float smem[];
  const int bid = blockIdx.x;
  const int tid = threadIdx.x;
  const Smem S = carve(smem, a);
  const Prob P = prob_of(a, bid);
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  for (int j = tid; j < n; j += NT) S.x[j] = a.x[(long long)bid * n + j];
  for (int l = tid; l < m; l += NT) S.y[l] = a.y[(long long)bid * m + l];
  for (int k = tid; k < p; k += NT) {
    S.z[k] = a.z[(long long)bid * p + k];
    S.s[k] = a.s[(long long)bid * p + k];
  }
  __syncthreads();
  int status = (a.status[bid] & 0xff) == ST_CONVERGED ? ST_CONVERGED : (ST_FAIL | (STG_RELAX << 8));
  int it = 0;
  if (status == ST_CONVERGED) {
    float phi_prev = INFINITY;
    for (int k = 0;; ++k) {
      float kappa = manifold_coords<NT>(S, a);
      const Norms R = residuals<NT>(S, a, P, kappa, kappa - a.kappa_relax);
      const float dmax = assemble<NT>(S, a, P, S.dp, S.dp, S.dm, false, false);
      factor_qd<NT>(S.K, a.kl, a.floor_rel * dmax, S.rinv, S.flag);
      it = k;
      if (R.nonfin > 0.f) { status = ST_FAIL | (STG_RELAX << 8); break; }
      const bool kok = p == 0 || fabsf(kappa / a.kappa_relax - 1.f) <= a.relax_ktol;
      if (kok && relax_done(R, a.tol, a.relax_tol, phi_prev)) break;
      phi_prev = kok ? rel_phi(R) : INFINITY;
      if (k == a.relax_max_iter) { status = ST_MAX_ITER | (STG_RELAX << 8); break; }
      solve_qd<NT>(S.K, a.kl, S.rinv, S.rhs);
      int stage = 0;
      if (!newton_update<NT>(S, a, P, kappa, kappa - a.kappa_relax, &stage)) {
        status = ST_FAIL | (STG_RELAX << 8);
        break;
      }
    }
  }
  // ---- Algorithm 3: M (dx, w, dy) = (−∇ₓℓ, 0, 0), dv = G dx + w, dz = d₊ ⊙ dv
  bool ok = status == ST_CONVERGED;
  if (ok) {
    for (int j = tid; j < a.N4; j += NT) S.rhs[j] = j < n ? -__ldg(a.dl + (long long)bid * n + j) : 0.f;
    __syncthreads();
    solve_qd<NT>(S.K, a.kl, S.rinv, S.rhs);
    rowdots<NT>(P.G, p, n, S.rhs, [&](int k, float gdx) { S.dz[k] = S.dp[k] * (gdx + S.rhs[n4 + k]); });
    for (int j = tid; j < n; j += NT) S.dx[j] = S.rhs[j];
    for (int l = tid; l < m; l += NT) S.dy[l] = S.rhs[n4 + p + l];
    __syncthreads();
    float bad = 0.f;
    for (int j = tid; j < n; j += NT) if (!isfinite(S.dx[j])) bad = 1.f;
    for (int k = tid; k < p; k += NT) if (!isfinite(S.dz[k])) bad = 1.f;
    for (int l = tid; l < m; l += NT) if (!isfinite(S.dy[l])) bad = 1.f;
    float v[1] = {bad};
    block_reduce<NT, 0, 1>(v, S.red);
    if (v[0] > 0.f) { ok = false; status = ST_FAIL | (STG_BACKWARD << 8); }
  }
  if (!ok) {  // zero-filled gradients for failed problems
    for (int j = tid; j < n; j += NT) { S.dx[j] = 0.f; S.x[j] = 0.f; }
    for (int l = tid; l < m; l += NT) { S.dy[l] = 0.f; S.y[l] = 0.f; }
    for (int k = tid; k < p; k += NT) { S.dz[k] = 0.f; S.z[k] = 0.f; }
    __syncthreads();
  }
  // ---- parameter gradients (coalesced stores)
  const long long bb = bid;
  if (a.gQ) {
    float* o = a.gQ + bb * n * n;
    for (int e = tid; e < n * n; e += NT) {
      const int i = e / n, j = e - i * n;
      o[e] = 0.5f * (S.dx[i] * S.x[j] + S.x[i] * S.dx[j]);
    }
  }
  if (a.gq) for (int j = tid; j < n; j += NT) a.gq[bb * n + j] = S.dx[j];
  if (a.gA) {
    float* o = a.gA + bb * m * n;
    for (int e = tid; e < m * n; e += NT) {
      const int l = e / n, j = e - l * n;
      o[e] = S.dy[l] * S.x[j] + S.y[l] * S.dx[j];
    }
  }
  if (a.gb) for (int l = tid; l < m; l += NT) a.gb[bb * m + l] = -S.dy[l];
  if (a.gG) {
    float* o = a.gG + bb * p * n;
    for (int e = tid; e < p * n; e += NT) {
      const int k = e / n, j = e - k * n;
      o[e] = S.dz[k] * S.x[j] + S.z[k] * S.dx[j];
    }
  }
  if (a.gh) for (int k = tid; k < p; k += NT) a.gh[bb * p + k] = -S.dz[k];
  if (a.wx) {
    for (int j = tid; j < n; j += NT) { a.wx[bb * n + j] = S.x[j]; a.wdx[bb * n + j] = S.dx[j]; }
    for (int l = tid; l < m; l += NT) { a.wy[bb * m + l] = S.y[l]; a.wdy[bb * m + l] = S.dy[l]; }
    for (int k = tid; k < p; k += NT) { a.wz[bb * p + k] = S.z[k]; a.wdz[bb * p + k] = S.dz[k]; }
  }
  if (tid == 0) {
    if (a.riters) a.riters[bid] = it;
    if (a.rstatus) a.rstatus[bid] = status;
  }
}

// ------------------------------------------------------------------------
// Batch sums for shared parameters (K8 of SURVEY §2.4; Alg. 3 formulas summed
// over the batch):  out[r][c] = scale · Σ_b (U[b][r] V[b][c] + U2[b][r] V2[b][c])
// 64×64 output tile per CTA, 256 threads, 4×4 outputs per thread; the batch
// dimension is staged through shared memory 32 rows at a time.
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) outer_sum_kernel(const float* __restrict__ U, const float* __restrict__ V,
                                                        const float* __restrict__ U2, const float* __restrict__ V2,
                                                        int B, int R, int Cc, float scale, float* __restrict__ out) {
  __shared__ float su[2][32][64], sv[2][32][64];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  float acc[4][4] = {};
  for (int b0 = 0; b0 < B; b0 += 32) {
    for (int e = tid; e < 32 * 64; e += 256) {
      const int bb = e >> 6, k = e & 63;
      const int b = b0 + bb;
      const bool okb = b < B;
      su[0][bb][k] = (okb && r0 + k < R) ? U[(long long)b * R + r0 + k] : 0.f;
      sv[0][bb][k] = (okb && c0 + k < Cc) ? V[(long long)b * Cc + c0 + k] : 0.f;
      su[1][bb][k] = (okb && r0 + k < R) ? U2[(long long)b * R + r0 + k] : 0.f;
      sv[1][bb][k] = (okb && c0 + k < Cc) ? V2[(long long)b * Cc + c0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int bb = 0; bb < 32; ++bb) {
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        float u[4], v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { u[i] = su[w][bb][tr + 16 * i]; v[i] = sv[w][bb][tc + 16 * i]; }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(u[i], v[j], acc[i][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = r0 + tr + 16 * i, c = c0 + tc + 16 * j;
      if (r < R && c < Cc) out[(long long)r * Cc + c] = scale * acc[i][j];
    }
}

// out[c] = scale · Σ_b U[b][c]
__global__ void __launch_bounds__(256) col_sum_kernel(const float* __restrict__ U, int B, int Cc, float scale,
                                                      float* __restrict__ out) {
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c >= Cc) return;
  float acc = 0.f;
  for (int b = 0; b < B; ++b) acc += U[(long long)b * Cc + c];
  out[c] = scale * acc;
}

}  // namespace qpb

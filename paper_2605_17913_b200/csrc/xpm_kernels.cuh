// xpm_kernels.cuh — the standard ("explicit") formulation, the comparison arm
// of config 3 (BASELINE.json: "standard vs bounded formulation in f32";
// SURVEY §8(a) row a13).  Reading Q18: Mehrotra
// predictor-corrector on the partially condensed system Eq. 8
// through the normal equations H = Q + Gᵀ D(z/s) G (+ the A-Schur block),
// factored WITHOUT a pivot floor so that a breakdown surfaces as a non-finite
// value (the failure the paper counts); relaxation by
// centering at κ_relax; adjoint (Q + GᵀD(z/s)G) dx + Aᵀdy = −∇ₓℓ, A dx = 0,
// dz = D(z/s) G dx, then Alg. 3's formulas.  Same CTA-per-QP machinery as the
// implicit kernels (assemble with all constraints condensed, factor_qd,
// solve_qd).
#pragma once
#include "ipm_kernels.cuh"

namespace qpb {

// out[j] = Σ_k Mat[k][j] vec[k]  (thread per column; Mat global rows×n)
template <int NT>
__device__ __noinline__ void coldots(const float* __restrict__ Mat, int rows, int n, const float* vec, float* out) {
  for (int j = threadIdx.x; j < n; j += NT) {
    float acc = 0.f;
    for (int k = 0; k < rows; ++k) acc = fmaf(__ldg(Mat + k * n + j), vec[k], acc);
    out[j] = acc;
  }
  __syncthreads();
}

// Eq. 4 residuals for the standard form; r_t → S.dx, r_i → S.rz, r_e → S.dy,
// Gx → S.gx, w = z/s → S.om.  Norms as in the implicit kernels (nrzs = 0).
template <int NT>
__device__ Norms x_residuals(const Smem& S, const Args& a, const Prob& P) {
  const int tid = threadIdx.x;
  const int n = a.n, p = a.p, m = a.m;
  rowdots<NT>(P.G, p, n, S.x, S.gx);
  rowdots<NT>(P.A, m, n, S.x, S.gx + p);
  float mri = 0.f, mgx = 0.f, ms = 0.f, mh = 0.f, mz = 0.f, gap = 0.f, nonfin = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float gx = S.gx[k], sk = S.s[k], zk = S.z[k], hk = __ldg(P.h + k);
    const float ri = gx + sk - hk;
    S.rz[k] = ri;
    S.om[k] = zk / sk;
    mri = fmaxf(mri, fabsf(ri)); mgx = fmaxf(mgx, fabsf(gx)); ms = fmaxf(ms, fabsf(sk));
    mh = fmaxf(mh, fabsf(hk)); mz = fmaxf(mz, fabsf(zk));
    gap = fmaf(sk, zk, gap);
    if (!isfinite(ri) || !isfinite(S.om[k])) nonfin += 1.f;
  }
  float mre = 0.f, max_ = 0.f, mb = 0.f;
  for (int l = tid; l < m; l += NT) {
    const float ax = S.gx[p + l], bl = __ldg(P.b + l);
    S.dy[l] = ax - bl;
    mre = fmaxf(mre, fabsf(ax - bl)); max_ = fmaxf(max_, fabsf(ax)); mb = fmaxf(mb, fabsf(bl));
  }
  float mrt = 0.f, mqx = 0.f, mq = 0.f, mgz = 0.f, may = 0.f, obj = 0.f;
  for (int j = tid; j < n; j += NT) {
    float qx = 0.f, gz = 0.f, ay = 0.f;
    for (int i = 0; i < n; ++i) qx = fmaf(__ldg(P.Q + i * n + j), S.x[i], qx);
    for (int k = 0; k < p; ++k) gz = fmaf(__ldg(P.G + k * n + j), S.z[k], gz);
    for (int l = 0; l < m; ++l) ay = fmaf(__ldg(P.A + l * n + j), S.y[l], ay);
    const float qj = __ldg(P.q + j);
    const float rt = qx + qj + gz + ay;
    S.dx[j] = rt;
    mrt = fmaxf(mrt, fabsf(rt)); mqx = fmaxf(mqx, fabsf(qx)); mq = fmaxf(mq, fabsf(qj));
    mgz = fmaxf(mgz, fabsf(gz)); may = fmaxf(may, fabsf(ay));
    obj = fmaf(S.x[j], fmaf(0.5f, qx, qj), obj);
    if (!isfinite(rt)) nonfin += 1.f;
  }
  float v[17] = {gap, obj, nonfin, mrt, mre, mri, 0.f, mqx, mq, mgz, may, max_, mb, mgx, ms, mh, mz};
  block_reduce<NT, 3, 14>(v, S.red);
  Norms R;
  R.gap = v[0]; R.obj = v[1]; R.nonfin = v[2]; R.nrt = v[3]; R.nre = v[4]; R.nri = v[5]; R.nrzs = 0.f;
  R.sQx = v[7]; R.sq = v[8]; R.sGz = v[9]; R.sAy = v[10]; R.sAx = v[11]; R.sb = v[12]; R.sGx = v[13];
  R.ss = v[14]; R.sh = v[15]; R.sz = v[16];
  R.pa = 0;
  return R;
}

// One Eq. 8 solve with the current factor for complementarity residual rc
// (in S.t): u = r_i − rc/z, rhs = (−r_t − Gᵀ(w⊙u), −r_e);  Δz = w⊙(GΔx + u),
// Δs = −(rc + s⊙Δz)/z.  Δx → dxo, Δy → dyo, Δz → dzo, Δs → dso.  Returns
// false if a component is not finite.
template <int NT>
__device__ bool x_direction(const Smem& S, const Args& a, const Prob& P, float* K, const KLayout& L, float* dxo,
                            float* dyo, float* dzo, float* dso) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  for (int k = tid; k < p; k += NT) {
    const float u = S.rz[k] - S.t[k] / S.z[k];
    S.f2[k] = u;
    S.c[k] = S.om[k] * u;
  }
  __syncthreads();
  coldots<NT>(P.G, p, n, S.c, S.rhs);  // Gᵀ(w⊙u) into rhs[0:n]
  for (int j = tid; j < n4; j += NT) S.rhs[j] = j < n ? -S.dx[j] - S.rhs[j] : 0.f;
  for (int l = tid; l < m; l += NT) S.rhs[n4 + l] = -S.dy[l];
  for (int j = L.N + tid; j < L.N4; j += NT) S.rhs[j] = 0.f;
  __syncthreads();
  solve_qd<NT>(K, L, S.rinv, S.rhs);
  rowdots<NT>(P.G, p, n, S.rhs, S.gx);
  float bad = 0.f;
  for (int k = tid; k < p; k += NT) {
    const float dz = S.om[k] * (S.gx[k] + S.f2[k]);
    const float ds = -(S.t[k] + S.s[k] * dz) / S.z[k];
    dzo[k] = dz; dso[k] = ds;
    if (!isfinite(dz) || !isfinite(ds)) bad = 1.f;
  }
  for (int j = tid; j < n; j += NT) { dxo[j] = S.rhs[j]; if (!isfinite(S.rhs[j])) bad = 1.f; }
  for (int l = tid; l < m; l += NT) { dyo[l] = S.rhs[n4 + l]; if (!isfinite(S.rhs[n4 + l])) bad = 1.f; }
  float v[1] = {bad};
  block_reduce<NT, 0, 1>(v, S.red);
  return !(v[0] > 0.f);
}

// α_max of Eq. 6 over (s, z) + (ds, dz) (block-uniform)
template <int NT>
__device__ float x_alpha_max(const Smem& S, int p, const float* dz, const float* ds) {
  float am = INFINITY;
  for (int k = threadIdx.x; k < p; k += NT) {
    if (ds[k] < 0.f) am = fminf(am, -S.s[k] / ds[k]);
    if (dz[k] < 0.f) am = fminf(am, -S.z[k] / dz[k]);
  }
  return block_min<NT>(am, S.red + 64);
}

// CVXOPT initialisation, as in the implicit solve kernel.
template <int NT>
__device__ bool x_init(const Smem& S, const Args& a, const Prob& P) {
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  for (int i = tid; i < p; i += NT) S.om[i] = 1.f;
  __syncthreads();
  const KLayout L = KLayout::make(n4 + m, n4);
  const float dmax = assemble<NT>(S.K, S, a, P, L, 0, S.om, S.om, S.om);
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
  factor_qd<NT>(S.K, L, a.floor_rel * dmax, S.rinv, S.flag, S.scr);
  solve_qd<NT>(S.K, L, S.rinv, S.rhs);
  for (int j = tid; j < n; j += NT) S.x[j] = S.rhs[j];
  for (int l = tid; l < m; l += NT) S.y[l] = S.rhs[n4 + l];
  __syncthreads();
  rowdots<NT>(P.G, p, n, S.x, S.dz);
  float ap = -INFINITY, ad = -INFINITY, bad = 0.f;
  for (int i = tid; i < p; i += NT) {
    const float zh = S.dz[i] - __ldg(P.h + i);
    S.dz[i] = zh;
    ap = fmaxf(ap, zh); ad = fmaxf(ad, -zh);
    if (!isfinite(zh)) bad = 1.f;
  }
  for (int j = tid; j < n; j += NT) if (!isfinite(S.x[j])) bad = 1.f;
  float v[3] = {ap, ad, bad};
  block_reduce<NT, 0, 3>(v, S.red);
  for (int i = tid; i < p; i += NT) {
    const float zh = S.dz[i];
    S.s[i] = v[0] >= 0.f ? -zh + (1.f + v[0]) : -zh;
    S.z[i] = v[1] >= 0.f ? zh + (1.f + v[1]) : zh;
  }
  __syncthreads();
  return !(v[2] > 0.f);
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) xpm_solve_kernel(const Args a) {
  extern __shared__ __align__(16) float smem[];
  const Smem S = carve(smem, a);
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  // predictor directions live in rinv-free scratch: Δx_a → S.dz? no: dedicated views
  float* dxa = S.ds_x;
  for (int bid = blockIdx.x; bid < a.B; bid += gridDim.x) {
    const Prob P = prob_of(a, bid);
    int status = ST_CONVERGED, it = 0;
    float fl = 0.f;
    if (!x_init<NT>(S, a, P)) status = ST_FAIL | (STG_INIT << 8);
    const KLayout L = KLayout::make(n4 + m, n4);
    for (int k = 0; status == ST_CONVERGED; ++k) {
      const Norms R = x_residuals<NT>(S, a, P);
      it = k;
      fl += iter_flops(n, m, p, 0, true, false, false);
      if (R.nonfin > 0.f) { status = ST_FAIL | (STG_SCALING << 8); break; }
      if (converged_solve(R, a.tol)) break;
      if (k == a.max_iter) { status = ST_MAX_ITER; break; }
      const float mu = R.gap / (float)p;
      const float dmax = assemble<NT>(S.K, S, a, P, L, 0, S.om, S.om, S.om);
      factor_qd<NT>(S.K, L, 0.f * dmax, S.rinv, S.flag, S.scr);  // no pivot floor (Q18)
      fl += iter_flops(n, m, p, 0, false, true, true) + 2.f * L.N * L.N + 4.f * p * n;
      // affine predictor: r_c = z ⊙ s
      for (int i = tid; i < p; i += NT) S.t[i] = S.z[i] * S.s[i];
      __syncthreads();
      if (!x_direction<NT>(S, a, P, S.K, L, dxa, dxa + n4, S.dp, S.dm)) { status = ST_FAIL | (STG_PREDICTOR << 8); break; }
      const float aa = fminf(1.f, x_alpha_max<NT>(S, p, S.dp, S.dm));
      float mua = 0.f;
      for (int i = tid; i < p; i += NT) mua += (S.s[i] + aa * S.dm[i]) * (S.z[i] + aa * S.dp[i]);
      float v1[1] = {mua};
      block_reduce<NT, 1, 0>(v1, S.red);
      const float ratio = v1[0] / (float)p / mu;
      const float sig = ratio * ratio * ratio;  // σ = (μ_aff/μ)³
      if (!isfinite(sig) || !isfinite(mu)) { status = ST_FAIL | (STG_CENTERING << 8); break; }
      // corrector: r_c = z ⊙ s + Δs_a ⊙ Δz_a − σ μ
      for (int i = tid; i < p; i += NT) S.t[i] = S.z[i] * S.s[i] + S.dm[i] * S.dp[i] - sig * mu;
      __syncthreads();
      if (!x_direction<NT>(S, a, P, S.K, L, S.dx, S.dy, S.dz, S.v)) { status = ST_FAIL | (STG_CORRECTOR << 8); break; }
      const float alpha = fminf(1.f, a.tau * x_alpha_max<NT>(S, p, S.dz, S.v));
      if (!(alpha > 0.f) || !isfinite(alpha)) { status = ST_FAIL | (STG_LINESEARCH << 8); break; }
      for (int j = tid; j < n; j += NT) S.x[j] = fmaf(alpha, S.dx[j], S.x[j]);
      for (int l = tid; l < m; l += NT) S.y[l] = fmaf(alpha, S.dy[l], S.y[l]);
      for (int i = tid; i < p; i += NT) {
        S.z[i] = fmaf(alpha, S.dz[i], S.z[i]);
        S.s[i] = fmaf(alpha, S.v[i], S.s[i]);
      }
      __syncthreads();
    }
    for (int j = tid; j < n; j += NT) a.x[(long long)bid * n + j] = S.x[j];
    for (int l = tid; l < m; l += NT) a.y[(long long)bid * m + l] = S.y[l];
    for (int i = tid; i < p; i += NT) {
      a.z[(long long)bid * p + i] = S.z[i];
      a.s[(long long)bid * p + i] = S.s[i];
    }
    if (tid == 0) {
      a.iters[bid] = it;
      a.status[bid] = status;
      if (a.flops) a.flops[bid] = fl;
    }
    __syncthreads();
  }
}

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) xpm_backward_kernel(const Args a) {
  extern __shared__ __align__(16) float smem[];
  const Smem S = carve(smem, a);
  const int tid = threadIdx.x;
  const int n = a.n, n4 = a.n4, p = a.p, m = a.m;
  const KLayout L = KLayout::make(n4 + m, n4);
  float* ddx = S.ds_x;  // centering direction Δx (n4) and Δy (m4)
  for (int bid = blockIdx.x; bid < a.B; bid += gridDim.x) {
    const Prob P = prob_of(a, bid);
    for (int j = tid; j < n; j += NT) S.x[j] = a.x[(long long)bid * n + j];
    for (int l = tid; l < m; l += NT) S.y[l] = a.y[(long long)bid * m + l];
    for (int i = tid; i < p; i += NT) {
      S.z[i] = a.z[(long long)bid * p + i];
      S.s[i] = a.s[(long long)bid * p + i];
    }
    __syncthreads();
    int status = (a.status[bid] & 0xff) == ST_CONVERGED ? ST_CONVERGED : (ST_FAIL | (STG_RELAX << 8));
    int it = 0;
    bool ok = false;
    float fl = 0.f;
    float phi_prev = INFINITY;
    for (int k = 0; status == ST_CONVERGED; ++k) {
      const Norms R = x_residuals<NT>(S, a, P);
      const float dmax = assemble<NT>(S.K, S, a, P, L, 0, S.om, S.om, S.om);
      factor_qd<NT>(S.K, L, 0.f * dmax, S.rinv, S.flag, S.scr);
      fl += iter_flops(n, m, p, 0, true, true, true);
      it = k;
      if (R.nonfin > 0.f) { status = ST_FAIL | (STG_RELAX << 8); break; }
      float dev = 0.f;
      for (int i = tid; i < p; i += NT) dev = fmaxf(dev, fabsf(S.z[i] * S.s[i] / a.kappa_relax - 1.f));
      float vd[1] = {dev};
      block_reduce<NT, 0, 1>(vd, S.red);
      const bool kok = p == 0 || vd[0] <= a.relax_ktol;
      const bool done = kok && relax_done(R, a.tol, a.relax_tol, phi_prev);
      phi_prev = kok ? rel_phi(R) : INFINITY;
      if (!done && k == a.relax_max_iter) { status = ST_MAX_ITER | (STG_RELAX << 8); break; }
      if (done) {
        // adjoint: (Q + GᵀWG) dx + Aᵀdy = −∇ₓℓ, A dx = 0, dz = W G dx
        for (int j = tid; j < L.N4; j += NT) S.rhs[j] = j < n ? -__ldg(a.dl + (long long)bid * n + j) : 0.f;
        __syncthreads();
        solve_qd<NT>(S.K, L, S.rinv, S.rhs);
        rowdots<NT>(P.G, p, n, S.rhs, S.gx);
        for (int i = tid; i < p; i += NT) S.dz[i] = S.om[i] * S.gx[i];
        for (int j = tid; j < n; j += NT) S.dx[j] = S.rhs[j];
        for (int l = tid; l < m; l += NT) S.dy[l] = S.rhs[n4 + l];
        __syncthreads();
        float bad = 0.f;
        for (int j = tid; j < n; j += NT) if (!isfinite(S.dx[j])) bad = 1.f;
        for (int i = tid; i < p; i += NT) if (!isfinite(S.dz[i])) bad = 1.f;
        float vb[1] = {bad};
        block_reduce<NT, 0, 1>(vb, S.red);
        ok = !(vb[0] > 0.f);
        if (!ok) status = ST_FAIL | (STG_BACKWARD << 8);
        break;
      }
      // centering step: r_c = z ⊙ s − κ_relax
      for (int i = tid; i < p; i += NT) S.t[i] = S.z[i] * S.s[i] - a.kappa_relax;
      __syncthreads();
      if (!x_direction<NT>(S, a, P, S.K, L, ddx, ddx + n4, S.dp, S.dm)) { status = ST_FAIL | (STG_RELAX << 8); break; }
      const float alpha = fminf(1.f, a.tau * x_alpha_max<NT>(S, p, S.dp, S.dm));
      for (int j = tid; j < n; j += NT) S.x[j] = fmaf(alpha, ddx[j], S.x[j]);
      for (int l = tid; l < m; l += NT) S.y[l] = fmaf(alpha, ddx[n4 + l], S.y[l]);
      for (int i = tid; i < p; i += NT) {
        S.z[i] = fmaf(alpha, S.dp[i], S.z[i]);
        S.s[i] = fmaf(alpha, S.dm[i], S.s[i]);
      }
      __syncthreads();
    }
    if (!ok) {
      for (int j = tid; j < n; j += NT) { S.dx[j] = 0.f; S.x[j] = 0.f; }
      for (int l = tid; l < m; l += NT) { S.dy[l] = 0.f; S.y[l] = 0.f; }
      for (int i = tid; i < p; i += NT) { S.dz[i] = 0.f; S.z[i] = 0.f; }
      __syncthreads();
    }
    write_gradients<NT>(S, a, bid);
    if (tid == 0) {
      if (a.riters) a.riters[bid] = it;
      if (a.rstatus) a.rstatus[bid] = status;
      if (a.flops) a.flops[bid] = fl + 2.f * (n * n + m * n + p * n);
    }
    __syncthreads();
  }
}

}  // namespace qpb

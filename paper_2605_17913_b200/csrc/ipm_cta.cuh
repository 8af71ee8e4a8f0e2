// ipm_cta.cuh — CTA-level building blocks of the persistent per-problem IPM
// kernel (one CTA owns one QP; its KKT matrix stays resident in shared memory
// for the whole of Alg. 1, or of Alg. 2 + Alg. 3).
//
// KKT layout: the bounded system of Eq. 14 is
// factored in its congruent quasi-definite form (reading Q12)
//       M = [[Q + Gᵀ D₊ G,  Gᵀ D₊,  Aᵀ],
//            [D₊ G,         −D₋,    0 ],
//            [A,            0,      0 ]]      unknowns (Δx, w, Δy), Δv = GΔx + w
// with D₊ = diag(∂b_κ(v)), D₋ = diag(∂b_κ(−v)) ∈ (0,1] (Eq. 11).  Rows/cols:
//   x-block [0, n4)   (n4 = n rounded up to 4; padded rows are identity)
//   w-block [n4, n4+nw)
//   y-block [n4+nw, N)
// stored row-major, lower triangle, leading dimension ld (ld/4 odd so that
// 16-byte accesses of 8 consecutive rows hit 8 distinct bank groups).
// Factorisation: M = L S Lᵀ, S = diag(+1 on the x-block, −1 elsewhere), a
// "signed Cholesky" that needs no pivoting because M is quasi-definite.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace qpb {

constexpr int KB = 16;  // panel width of the blocked factorisation / solves

// ------------------------------------------------------------------------
// Retraction map, App. C, written for f32 on the device.
//   b_κ(v)   = (v + √(v²+4κ))/2            v ≥ 0
//            = 2κ / (√(v²+4κ) − v)         v < 0
//   ∂b_κ(v)  = ½ (1 + v/√(v²+4κ))          v ≥ 0
//            = 2κ / (v²+4κ − v√(v²+4κ))    v < 0
//   ∂_κ b_κ  = 1/√(v²+4κ)                  (reading Q10)
// ------------------------------------------------------------------------
__device__ __forceinline__ float ret_b(float v, float k) {
  const float R2 = v * v + 4.f * k;
  const float R = sqrtf(R2);
  return v >= 0.f ? 0.5f * (v + R) : (2.f * k) / (R - v);
}
__device__ __forceinline__ float ret_db(float v, float k) {
  const float R2 = v * v + 4.f * k;
  const float R = sqrtf(R2);
  return v >= 0.f ? 0.5f * (1.f + v / R) : (2.f * k) / (R2 - v * R);
}
__device__ __forceinline__ float ret_dk(float v, float k) { return 1.f / sqrtf(v * v + 4.f * k); }

__device__ __forceinline__ int r4(int x) { return (x + 3) & ~3; }

// Panel boundaries: width KB, never straddling npos (so the sign is uniform
// inside a panel).
__device__ __forceinline__ int panel_end(int k0, int N, int npos) {
  int k1 = min(k0 + KB, N);
  if (k0 < npos) k1 = min(k1, npos);
  return k1;
}
__device__ __forceinline__ int last_panel_start(int N, int npos) {
  if (N > npos) return npos + ((N - 1 - npos) / KB) * KB;
  return ((N - 1) / KB) * KB;
}
__device__ __forceinline__ int prev_panel_start(int k0, int npos) {
  // panel preceding the one starting at k0 (k0 > 0)
  if (k0 > npos) return k0 - KB;
  // k0 == npos (or k0 inside the x-block, which is KB-aligned)
  if (k0 == npos) return ((npos - 1) / KB) * KB;
  return k0 - KB;
}

// ------------------------------------------------------------------------
// Block reductions: NS sums followed by NM maxima, fixed order (deterministic).
// Every thread returns the reduced values.  `red` is a shared scratch of at
// least (NT/32)*(NS+NM) floats.
// ------------------------------------------------------------------------
template <int NT, int NS, int NM>
__device__ __forceinline__ void block_reduce(float (&v)[NS + NM], float* red) {
  constexpr int NW = NT / 32, NV = NS + NM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a = v[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float b = __shfl_xor_sync(0xffffffffu, a, o);
      a = (i < NS) ? a + b : fmaxf(a, b);
    }
    v[i] = a;
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp * NV + i] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float a = red[i];
#pragma unroll
    for (int w = 1; w < NW; ++w) a = (i < NS) ? a + red[w * NV + i] : fmaxf(a, red[w * NV + i]);
    v[i] = a;
  }
}

template <int NT>
__device__ __forceinline__ float block_min(float a, float* red) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) a = fminf(a, __shfl_xor_sync(0xffffffffu, a, o));
  __syncthreads();
  if (lane == 0) red[warp] = a;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) r = fminf(r, red[w]);
  return r;
}

// ------------------------------------------------------------------------
// Signed Cholesky (quasi-definite LDLᵀ) of the N×N lower triangle held in
// K (leading dimension ld, N4 = r4(N) rows allocated, rows ≥ N zero).
// Pivots k < npos must be positive, k ≥ npos negative; a pivot on the wrong
// side of ±θ is replaced by ±θ (reading Q12) and counted.  On exit the lower
// triangle holds L with M = L S Lᵀ and rinv[k] = 1/L[k][k].
// Right-looking, panel width KB:
//   (a) warp 0 factors the kb×kb diagonal block in registers (shuffles);
//   (b) every thread solves one row of the panel below (TRSM);
//   (c) the trailing lower triangle takes the rank-kb update (SYRK) in 32×32
//       super-tiles, 64 threads per super-tile, 4×4 strided register tiles.
// Returns the number of floored pivots (block-uniform).
// ------------------------------------------------------------------------
template <int NT>
__device__ int factor_qd(float* __restrict__ K, const int ld, const int N, const int N4, const int npos,
                         const float theta, float* __restrict__ rinv, int* __restrict__ flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int nfloor = 0;
  for (int k0 = 0; k0 < N;) {
    const int k1 = panel_end(k0, N, npos);
    const int kb = k1 - k0;
    const float sgn = k0 < npos ? 1.f : -1.f;
    // ---- (a) diagonal block -------------------------------------------------
    if (warp == 0) {
      float a[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) a[j] = (lane < kb && j < kb) ? K[(k0 + lane) * ld + k0 + j] : 0.f;
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        if (k < kb) {
          float d = sgn * __shfl_sync(0xffffffffu, a[k], k);
          if (!(d >= theta)) { d = theta; ++nfloor; }
          const float l = sqrtf(d);
          const float ri = 1.f / l;
          if (lane == k) a[k] = l;
          else if (lane > k) a[k] *= sgn * ri;  // l_rk = a_rk / (s_k l_kk)
          if (lane == 0) rinv[k0 + k] = ri;
#pragma unroll
          for (int j = k + 1; j < KB; ++j) {
            const float ljk = __shfl_sync(0xffffffffu, a[k], j);
            if (j < kb && lane >= j) a[j] = fmaf(-sgn * a[k], ljk, a[j]);
          }
        }
      }
      if (lane < kb) {
#pragma unroll
        for (int j = 0; j < KB; ++j)
          if (j <= lane) K[(k0 + lane) * ld + k0 + j] = a[j];
      }
    }
    __syncthreads();
    // ---- (b) panel rows below the diagonal block: x L11ᵀ = a, l = s·x -------
    for (int i = k1 + tid; i < N; i += NT) {
      float a[KB];
      const float4* row = reinterpret_cast<const float4*>(K + i * ld + k0);
#pragma unroll
      for (int j4 = 0; j4 < KB / 4; ++j4) {
        float4 t = (4 * j4 < kb) ? row[j4] : make_float4(0.f, 0.f, 0.f, 0.f);
        a[4 * j4] = t.x; a[4 * j4 + 1] = t.y; a[4 * j4 + 2] = t.z; a[4 * j4 + 3] = t.w;
      }
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        if (k < kb) {
          const float xk = a[k] * rinv[k0 + k];
          a[k] = xk;
#pragma unroll
          for (int j = k + 1; j < KB; ++j)
            if (j < kb) a[j] = fmaf(-xk, K[(k0 + j) * ld + k0 + k], a[j]);
        }
      }
      float4* wrow = reinterpret_cast<float4*>(K + i * ld + k0);
#pragma unroll
      for (int j4 = 0; j4 < KB / 4; ++j4)
        if (4 * j4 < kb)
          wrow[j4] = make_float4(sgn * a[4 * j4], sgn * a[4 * j4 + 1], sgn * a[4 * j4 + 2], sgn * a[4 * j4 + 3]);
    }
    __syncthreads();
    // ---- (c) trailing update A22 -= s · L21 L21ᵀ (lower super-tiles) -------
    if (k1 < N) {
      const int T = (N4 - k1 + 31) >> 5;
      const int nst = T * (T + 1) / 2;
      const int grp = tid >> 6, gt = tid & 63, ty = gt >> 3, tx = gt & 7;
      const int kq = (kb + 3) >> 2;  // kb is a multiple of 4 except on a final panel (no trailing then)
      for (int st = grp; st < nst; st += NT / 64) {
        int I = (int)((sqrtf(8.f * st + 1.f) - 1.f) * 0.5f);
        while ((I + 1) * (I + 2) / 2 <= st) ++I;
        while (I * (I + 1) / 2 > st) --I;
        const int J = st - I * (I + 1) / 2;
        const int rb = k1 + 32 * I + ty, cb = k1 + 32 * J + tx;
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int r = rb + 8 * a, c = cb + 8 * b;
            acc[a][b] = (r < N4 && c < N4) ? K[r * ld + c] : 0.f;
          }
        for (int q = 0; q < kq; ++q) {
          float4 lr[4], lc[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int r = rb + 8 * a;
            lr[a] = r < N4 ? *reinterpret_cast<const float4*>(K + r * ld + k0 + 4 * q) : make_float4(0, 0, 0, 0);
          }
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int c = cb + 8 * b;
            float4 t = c < N4 ? *reinterpret_cast<const float4*>(K + c * ld + k0 + 4 * q) : make_float4(0, 0, 0, 0);
            t.x *= sgn; t.y *= sgn; t.z *= sgn; t.w *= sgn;
            lc[b] = t;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              float t = acc[a][b];
              t = fmaf(-lr[a].x, lc[b].x, t);
              t = fmaf(-lr[a].y, lc[b].y, t);
              t = fmaf(-lr[a].z, lc[b].z, t);
              t = fmaf(-lr[a].w, lc[b].w, t);
              acc[a][b] = t;
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int r = rb + 8 * a, c = cb + 8 * b;
            if (r < N4 && c < N4) K[r * ld + c] = acc[a][b];
          }
      }
    }
    __syncthreads();
    k0 = k1;
  }
  if (tid == 0) *flag = nfloor;
  __syncthreads();
  const int r = *flag;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------------
// Solve M u = rhs in place with the factor of factor_qd (M = L S Lᵀ).
// ------------------------------------------------------------------------
template <int NT>
__device__ void solve_qd(const float* __restrict__ K, const int ld, const int N, const int npos,
                         const float* __restrict__ rinv, float* __restrict__ rhs) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // forward: L u = b
  for (int k0 = 0; k0 < N;) {
    const int k1 = panel_end(k0, N, npos);
    const int kb = k1 - k0;
    if (warp == 0) {
      float Lr[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) Lr[j] = (lane < kb && j < lane) ? K[(k0 + lane) * ld + k0 + j] : 0.f;
      float bv = lane < kb ? rhs[k0 + lane] : 0.f;
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        if (k < kb) {
          const float uk = __shfl_sync(0xffffffffu, bv, k) * rinv[k0 + k];
          if (lane == k) bv = uk;
          else if (lane > k) bv = fmaf(-Lr[k], uk, bv);
        }
      }
      if (lane < kb) rhs[k0 + lane] = bv;
    }
    __syncthreads();
    for (int i = k1 + tid; i < N; i += NT) {
      const float4* row = reinterpret_cast<const float4*>(K + i * ld + k0);
      float acc = rhs[i];
      for (int j4 = 0; 4 * j4 < kb; ++j4) {
        const float4 l = row[j4];
        const int j = k0 + 4 * j4;
        acc = fmaf(-l.x, rhs[j], acc);
        if (4 * j4 + 1 < kb) acc = fmaf(-l.y, rhs[j + 1], acc);
        if (4 * j4 + 2 < kb) acc = fmaf(-l.z, rhs[j + 2], acc);
        if (4 * j4 + 3 < kb) acc = fmaf(-l.w, rhs[j + 3], acc);
      }
      rhs[i] = acc;
    }
    __syncthreads();
    k0 = k1;
  }
  // u <- S u
  for (int i = npos + tid; i < N; i += NT) rhs[i] = -rhs[i];
  __syncthreads();
  // backward: Lᵀ x = u, panels in reverse order
  for (int k0 = last_panel_start(N, npos);; k0 = prev_panel_start(k0, npos)) {
    const int k1 = panel_end(k0, N, npos);
    const int kb = k1 - k0;
    if (warp == 0) {
      float Lc[KB];  // lane j holds column j of the diagonal block
#pragma unroll
      for (int i = 0; i < KB; ++i) Lc[i] = (lane < kb && i < kb && i > lane) ? K[(k0 + i) * ld + k0 + lane] : 0.f;
      float bv = lane < kb ? rhs[k0 + lane] : 0.f;
#pragma unroll
      for (int k = KB - 1; k >= 0; --k) {
        if (k < kb) {
          const float xk = __shfl_sync(0xffffffffu, bv, k) * rinv[k0 + k];
          if (lane == k) bv = xk;
          else if (lane < k) bv = fmaf(-Lc[k], xk, bv);
        }
      }
      if (lane < kb) rhs[k0 + lane] = bv;
    }
    __syncthreads();
    for (int j = tid; j < k0; j += NT) {
      float acc = rhs[j];
      for (int i = 0; i < kb; ++i) acc = fmaf(-K[(k0 + i) * ld + j], rhs[k0 + i], acc);
      rhs[j] = acc;
    }
    __syncthreads();
    if (k0 == 0) break;
  }
}

}  // namespace qpb

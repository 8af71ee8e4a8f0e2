// ipm_cta.cuh — CTA-level building blocks of the persistent per-problem IPM
// kernel (one CTA owns one QP; its KKT matrix stays resident in shared memory
// for the whole of Alg. 1, or of Alg. 2 + Alg. 3).
//
// KKT matrix: the bounded system of Eq. 14 is
// factored in its congruent quasi-definite form (reading Q12)
//       M = [[Q + Gᵀ D₊ G,  Gᵀ D₊,  Aᵀ],
//            [D₊ G,         −D₋,    0 ],
//            [A,            0,      0 ]]      unknowns (Δx, w, Δy), Δv = GΔx + w
// with D₊ = diag(∂b_κ(v)), D₋ = diag(∂b_κ(−v)) ∈ (0,1] (Eq. 11).  Rows/cols:
//   x-block [0, n4)   (n4 = n rounded up to 4; padded rows are +identity)
//   w-block [n4, n4+nw), y-block [n4+nw, N), padding [N, N4) (−identity).
// Factorisation M = L S Lᵀ, S = diag(+1 on the x-block, −1 elsewhere): a
// "signed Cholesky" with no pivoting, valid because M is quasi-definite.
//
// Storage: packed lower triangle in 16-row blocks.  Row i of block b = i/16
// holds columns [0, 16(b+1)) (the whole diagonal block) plus 4 floats of
// padding, so that every row starts 16-byte aligned and consecutive rows are
// an ODD number of 16-byte units apart (8 consecutive rows read as float4 hit
// 8 distinct bank groups).  The last block may be partial (N4 not a multiple
// of 16).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace qpb {

constexpr int KB = 16;  // block / panel width

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

__host__ __device__ __forceinline__ int r4(int x) { return (x + 3) & ~3; }

// ------------------------------------------------------------------------
// Packed block layout of the lower triangle.
// ------------------------------------------------------------------------
struct KLayout {
  int N, N4, NB, npos;  // real dim, padded dim (×4), #16-blocks, #positive pivots
  int wl, Ll, baseL;    // last block: width, row length, offset
  __host__ __device__ static KLayout make(int N, int npos) {
    KLayout L;
    L.N = N;
    L.N4 = r4(N);
    L.NB = (L.N4 + KB - 1) / KB;
    L.npos = npos;
    L.wl = L.N4 - KB * (L.NB - 1);
    L.Ll = ((L.N4 >> 2) & 1) ? L.N4 : L.N4 + 4;
    const int b = L.NB - 1;
    L.baseL = 128 * b * (b + 1) + 64 * b;
    return L;
  }
  __host__ __device__ int size() const { return baseL + wl * Ll; }
  __host__ __device__ __forceinline__ int len(int b) const { return b < NB - 1 ? 16 * b + 20 : Ll; }
  __host__ __device__ __forceinline__ int off(int i) const {
    const int b = i >> 4, t = i & 15;
    return b < NB - 1 ? 128 * b * (b + 1) + 64 * b + t * (16 * b + 20) : baseL + t * Ll;
  }
  __host__ __device__ __forceinline__ int bw(int b) const { return b < NB - 1 ? KB : wl; }
};

__device__ __forceinline__ float sgn_of(int k, int npos) { return k < npos ? 1.f : -1.f; }

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
// Diagonal block factorisation by ONE warp: block b (width kb ≤ 16) of the
// packed matrix.  Lane r holds row r of the block in registers.  Step k: the
// pivot comes from lane k (its diagonal is already final), column k is
// scaled, and every lane updates its row; the next pivot only needs lane k+1's
// own l_{k+1,k}, so the critical chain per step is shfl → rsqrt → mul → fma.
// Returns the number of floored pivots (valid on every lane).
// ------------------------------------------------------------------------
__device__ __forceinline__ int factor_diag_block(float* __restrict__ K, const KLayout& L, int b, float theta,
                                                 float* __restrict__ rinv) {
  const int lane = threadIdx.x & 31;
  const int k0 = KB * b, kb = L.bw(b);
  float* row = K + L.off(k0 + (lane < kb ? lane : 0));
  float a[KB];
#pragma unroll
  for (int j4 = 0; j4 < KB / 4; ++j4) {
    float4 t = (lane < kb && 4 * j4 < kb) ? *reinterpret_cast<const float4*>(row + k0 + 4 * j4)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
    a[4 * j4] = t.x; a[4 * j4 + 1] = t.y; a[4 * j4 + 2] = t.z; a[4 * j4 + 3] = t.w;
  }
  int nfloor = 0;
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    if (k < kb) {
      const float s = sgn_of(k0 + k, L.npos);
      float d = s * __shfl_sync(0xffffffffu, a[k], k);
      if (!(d >= theta)) { d = theta; ++nfloor; }
      const float ri = rsqrtf(d);        // 1/l_kk
      const float l = d * ri;            // l_kk
      if (lane == k) a[k] = l;
      else if (lane > k) a[k] *= s * ri;  // l_rk = a_rk / (s_k l_kk)
      if (lane == 0) rinv[k0 + k] = ri;
      const float nl = -s * a[k];
#pragma unroll
      for (int j = k + 1; j < KB; ++j) {
        const float ljk = __shfl_sync(0xffffffffu, a[k], j);
        // lane j already holds l_jk: its own update (which feeds the next
        // pivot when j = k+1) does not wait for the shuffle
        if (lane == j) a[j] = fmaf(nl, a[k], a[j]);
        else if (lane > j) a[j] = fmaf(nl, ljk, a[j]);
      }
    }
  }
  if (lane < kb) {
#pragma unroll
    for (int j4 = 0; j4 < KB / 4; ++j4)
      if (4 * j4 < kb)
        *reinterpret_cast<float4*>(row + k0 + 4 * j4) = make_float4(a[4 * j4], a[4 * j4 + 1], a[4 * j4 + 2],
                                                                   a[4 * j4 + 3]);
  }
  return nfloor;
}

// ------------------------------------------------------------------------
// W = L_bb⁻¹ for a factored diagonal block, by ONE warp (lane c computes
// column c by forward substitution; L entries are broadcast reads).  The
// strict lower part of W is stored TRANSPOSED in the unused strict upper
// triangle of the diagonal block: W[r][c] (r > c) at row k0+c, column k0+r;
// diag(W) = rinv.  Used by solve_qd to turn the serial diagonal-block
// substitutions into 16×16 matrix-vector products.
// ------------------------------------------------------------------------
__device__ __forceinline__ void invert_diag_block(float* __restrict__ K, const KLayout& L, int b,
                                                  const float* __restrict__ rinv) {
  const int lane = threadIdx.x & 31;
  const int k0 = KB * b, kb = L.bw(b);
  const float* D = K + L.off(k0) + k0;
  const int Lb = L.len(b);
  float w[KB];
#pragma unroll
  for (int r = 0; r < KB; ++r) w[r] = 0.f;
  const int c = lane;
#pragma unroll
  for (int r = 0; r < KB; ++r) {
    if (r < kb) {
      // w_r = (δ_rc − Σ_{j<r} L[r][j] w_j) / L[r][r]; two partial sums shorten the chain
      float a0 = (r == c) ? 1.f : 0.f, a1 = 0.f;
#pragma unroll
      for (int j = 0; j < r; ++j) {
        const float l = D[r * Lb + j];
        if (j & 1) a1 = fmaf(-l, w[j], a1); else a0 = fmaf(-l, w[j], a0);
      }
      const float wr = (a0 + a1) * rinv[k0 + r];
      w[r] = (r >= c) ? wr : 0.f;
    }
  }
  if (c < kb) {
    float* rowc = K + L.off(k0 + c) + k0;
#pragma unroll
    for (int r = 0; r < KB; ++r)
      if (r > c && r < kb) rowc[r] = w[r];
  }
}

// ------------------------------------------------------------------------
// Signed Cholesky of the packed matrix K (layout L), right-looking with a
// depth-1 look-ahead, full 16-wide panels:
//   prologue: warp 0 factors diagonal block 0
//   for each block b with rows below it:
//     (1) TRSM   rows i ≥ 16(b+1):  x L_bbᵀ = a, l = S_b x         (thread per row)
//     (2) update block column b+1:  A[:, b+1] −= L[:, b] S_b L[b+1, b]ᵀ  (thread per row)
//     (3) warp 0 factors diagonal block b+1 WHILE warps 1.. apply the rank-16
//         update to the trailing lower triangle beyond block b+1 (32×32
//         super-tiles, one warp each, 8×4 strided register tiles).
// A pivot on the wrong side of ±θ is replaced by ±θ (reading Q12) and
// counted.  On exit K holds L (M = L S Lᵀ) and rinv[k] = 1/L[k][k].
// ------------------------------------------------------------------------
template <int NT>
__device__ int factor_qd(float* __restrict__ K, const KLayout& L, const float theta, float* __restrict__ rinv,
                         int* __restrict__ flag) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N4 = L.N4, npos = L.npos;
  int nfloor = 0;
  if (warp == 0) nfloor += factor_diag_block(K, L, 0, theta, rinv);
  __syncthreads();
  static_assert(NW >= 3, "factor_qd needs >= 3 warps");
  for (int b = 0; b + 1 < L.NB; ++b) {
    const int k0 = KB * b, r0 = k0 + KB;
    // ---- (1) TRSM of the panel rows below block b (full 16-wide panel) -------------
    for (int i = r0 + tid; i < N4; i += NT) {
      float* row = K + L.off(i) + k0;
      float a[KB];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 t = reinterpret_cast<const float4*>(row)[j4];
        a[4 * j4] = t.x; a[4 * j4 + 1] = t.y; a[4 * j4 + 2] = t.z; a[4 * j4 + 3] = t.w;
      }
      const float* D = K + L.off(k0) + k0;  // diagonal block: row j at D + j*Lb
      const int Lb = L.len(b);
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const float xk = a[k] * rinv[k0 + k];
        a[k] = xk;
#pragma unroll
        for (int j = k + 1; j < KB; ++j) a[j] = fmaf(-xk, D[j * Lb + k], a[j]);
      }
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float s0 = sgn_of(k0 + 4 * j4, npos);  // npos is a multiple of 4
        reinterpret_cast<float4*>(row)[j4] =
            make_float4(s0 * a[4 * j4], s0 * a[4 * j4 + 1], s0 * a[4 * j4 + 2], s0 * a[4 * j4 + 3]);
      }
    }
    __syncthreads();
    // ---- (2) look-ahead: block column b+1, rows i ≥ r0 -------------------------------
    const int w1 = L.bw(b + 1);
    const float* B1 = K + L.off(r0) + k0;  // rows of block b+1, panel columns of block b
    const int L1 = L.len(b + 1);
    for (int i = r0 + tid; i < N4; i += NT) {
      const float* li = K + L.off(i) + k0;
      float* ai = K + L.off(i) + r0;
      float lv[KB];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        float4 t = reinterpret_cast<const float4*>(li)[j4];
        const float s0 = sgn_of(k0 + 4 * j4, npos);
        lv[4 * j4] = s0 * t.x; lv[4 * j4 + 1] = s0 * t.y; lv[4 * j4 + 2] = s0 * t.z; lv[4 * j4 + 3] = s0 * t.w;
      }
#pragma unroll
      for (int c4 = 0; c4 < KB / 4; ++c4) {
        if (4 * c4 < w1) {
          float4 acc = reinterpret_cast<const float4*>(ai)[c4];
          float accv[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float* lj = B1 + (4 * c4 + cc) * L1;
            float t = accv[cc];
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const float4 u = reinterpret_cast<const float4*>(lj)[k4];
              t = fmaf(-lv[4 * k4], u.x, t);
              t = fmaf(-lv[4 * k4 + 1], u.y, t);
              t = fmaf(-lv[4 * k4 + 2], u.z, t);
              t = fmaf(-lv[4 * k4 + 3], u.w, t);
            }
            accv[cc] = t;
          }
          reinterpret_cast<float4*>(ai)[c4] = make_float4(accv[0], accv[1], accv[2], accv[3]);
        }
      }
    }
    __syncthreads();
    // ---- (3) warp 0: diagonal block b+1 ‖ warps 1..: trailing SYRK beyond block b+1 ----
    if (warp == 0) {
      nfloor += factor_diag_block(K, L, b + 1, theta, rinv);
    } else if (warp == 1) {
      invert_diag_block(K, L, b, rinv);
    } else {
      const int r2 = r0 + KB;
      if (r2 < N4) {
        const int T = (N4 - r2 + 31) >> 5;
        const int nst = T * (T + 1) / 2;
        const int ty = lane >> 3, tx = lane & 7;
        for (int st = warp - 2; st < nst; st += NW - 2) {
          int I = (int)((sqrtf(8.f * st + 1.f) - 1.f) * 0.5f);
          while ((I + 1) * (I + 2) / 2 <= st) ++I;
          while (I * (I + 1) / 2 > st) --I;
          const int J = st - I * (I + 1) / 2;
          const int rb = r2 + 32 * I + ty, cb = r2 + 32 * J + tx;
          int roff[8], coff[4];
          bool rok[8], cok[4];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            const int r = rb + 4 * a;
            rok[a] = r < N4;
            roff[a] = rok[a] ? L.off(r) : 0;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = cb + 8 * c;
            cok[c] = cc < N4;
            coff[c] = cok[c] ? L.off(cc) : 0;
          }
          float acc[8][4];
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][c] = (rok[a] && cok[c]) ? K[roff[a] + cb + 8 * c] : 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // S_b applied to the column operand (npos is a multiple of 4)
            const float sq = k0 + 4 * q < npos ? -1.f : 1.f;
            float4 lc[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float4 t = cok[c] ? *reinterpret_cast<const float4*>(K + coff[c] + k0 + 4 * q) : make_float4(0, 0, 0, 0);
              t.x *= sq; t.y *= sq; t.z *= sq; t.w *= sq;
              lc[c] = t;
            }
#pragma unroll
            for (int a = 0; a < 8; ++a) {
              const float4 lr = rok[a] ? *reinterpret_cast<const float4*>(K + roff[a] + k0 + 4 * q)
                                       : make_float4(0, 0, 0, 0);
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                float t = acc[a][c];
                t = fmaf(lr.x, lc[c].x, t);
                t = fmaf(lr.y, lc[c].y, t);
                t = fmaf(lr.z, lc[c].z, t);
                t = fmaf(lr.w, lc[c].w, t);
                acc[a][c] = t;
              }
            }
          }
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int cc = cb + 8 * c;
              // lower triangle only (the diagonal block's upper part is never touched)
              if (rok[a] && cok[c] && cc <= rb + 4 * a) K[roff[a] + cc] = acc[a][c];
            }
        }
      }
    }
    __syncthreads();
  }
  if (warp == 1) invert_diag_block(K, L, L.NB - 1, rinv);
  if (tid == 0) *flag = nfloor;
  __syncthreads();
  const int r = *flag;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------------
// Solve M u = rhs in place with the factor of factor_qd (M = L S Lᵀ), using
// the diagonal-block inverses W_b stored by invert_diag_block:
//   forward  (per block b):  u_b = W_b r_b;  r_i −= L_ib u_b for rows below
//   backward (per block b, last first):  x_b = W_bᵀ r_b;  r_j −= L_bjᵀ x_b above
// rhs has N4 entries (padding entries must be 0 on entry).
// ------------------------------------------------------------------------
template <int NT>
__device__ void solve_qd(const float* __restrict__ K, const KLayout& L, const float* __restrict__ rinv,
                         float* __restrict__ rhs) {
  const int tid = threadIdx.x;
  const int N4 = L.N4;
  // forward: L u = b
  for (int b = 0; b < L.NB; ++b) {
    const int k0 = KB * b, kb = L.bw(b);
    const float* D = K + L.off(k0) + k0;
    const int Lb = L.len(b);
    if (tid < 32) {
      const int t = tid;
      float r[KB];
#pragma unroll
      for (int c = 0; c < KB; ++c) r[c] = c < kb ? rhs[k0 + c] : 0.f;
      __syncwarp();
      if (t < kb) {
        float acc = rinv[k0 + t] * r[t];
#pragma unroll
        for (int c = 0; c < KB; ++c)
          if (c < t) acc = fmaf(D[c * Lb + t], r[c], acc);  // W[t][c] stored at row c, col t
        rhs[k0 + t] = acc;
      }
    }
    __syncthreads();
    if (b + 1 < L.NB) {
      const float4* u = reinterpret_cast<const float4*>(rhs + k0);
      for (int i = k0 + KB + tid; i < N4; i += NT) {
        const float4* row = reinterpret_cast<const float4*>(K + L.off(i) + k0);
        float acc = rhs[i];
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 l = row[j4], uu = u[j4];
          acc = fmaf(-l.x, uu.x, acc);
          acc = fmaf(-l.y, uu.y, acc);
          acc = fmaf(-l.z, uu.z, acc);
          acc = fmaf(-l.w, uu.w, acc);
        }
        rhs[i] = acc;
      }
      __syncthreads();
    }
  }
  // u <- S u
  for (int i = L.npos + tid; i < N4; i += NT) rhs[i] = -rhs[i];
  __syncthreads();
  // backward: Lᵀ x = u, blocks in reverse order
  for (int b = L.NB - 1; b >= 0; --b) {
    const int k0 = KB * b, kb = L.bw(b);
    const float* D = K + L.off(k0) + k0;
    const int Lb = L.len(b);
    if (tid < 32) {
      const int t = tid;
      float r[KB];
#pragma unroll
      for (int c = 0; c < KB; ++c) r[c] = c < kb ? rhs[k0 + c] : 0.f;
      __syncwarp();
      if (t < kb) {
        float acc = rinv[k0 + t] * r[t];
        const float* Dt = D + t * Lb;  // W[r][t] for r > t lives in row t, column r
#pragma unroll
        for (int c = 0; c < KB; ++c)
          if (c > t && c < kb) acc = fmaf(Dt[c], r[c], acc);
        rhs[k0 + t] = acc;
      }
    }
    __syncthreads();
    if (b > 0) {
      const float* Bk = K + L.off(k0);
      for (int j = tid; j < k0; j += NT) {
        float acc = rhs[j];
        for (int i = 0; i < kb; ++i) acc = fmaf(-Bk[i * Lb + j], rhs[k0 + i], acc);
        rhs[j] = acc;
      }
      __syncthreads();
    }
  }
}

}  // namespace qpb

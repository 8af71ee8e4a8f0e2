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
#ifndef QPB200_PANEL_COLS
#define QPB200_PANEL_COLS 2
#endif
constexpr int PC = QPB200_PANEL_COLS;  // panel columns per barrier (2 or 4)

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
  // uniform: the last block keeps the row length 16b + 20 of every other
  // block, so row offsets do not depend on N (the batched engine: one TMA
  // tensor map per 16-row block serves every problem and iteration)
  __host__ __device__ static KLayout make(int N, int npos, bool uniform = false) {
    KLayout L;
    L.N = N;
    L.N4 = r4(N);
    L.NB = (L.N4 + KB - 1) / KB;
    L.npos = npos;
    L.wl = L.N4 - KB * (L.NB - 1);
    L.Ll = uniform ? 16 * (L.NB - 1) + 20 : ((L.N4 >> 2) & 1) ? L.N4 : L.N4 + 4;
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

// Row offsets: from a shared-memory table (path 1 kernels fill it once per
// iteration; one LDS instead of the ~8-instruction formula in the hot loops)
// or from the formula.
template <bool TAB>
__device__ __forceinline__ int row_off(const KLayout& L, const int* __restrict__ tab, int i) {
  if constexpr (TAB) return tab[i];
  else return L.off(i);
}

__device__ __forceinline__ float sgn_of(int k, int npos) { return k < npos ? 1.f : -1.f; }

// Diagnostics (QPB200_PHASE_PROFILE): cycles spent by thread 0 in the
// factorisation sub-phases, summed over all CTAs: [panel, SYRK, inverses, count].
__device__ unsigned long long g_fac_cycles[4];
__device__ int g_fac_on;

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
// W = L_bb⁻¹ for a factored diagonal block, by ONE warp (lane c computes
// column c by forward substitution; L entries are broadcast reads).  The
// strict lower part of W is stored TRANSPOSED in the unused strict upper
// triangle of the diagonal block: W[r][c] (r > c) at row k0+c, column k0+r;
// diag(W) = rinv.  Used by solve_qd to turn the serial diagonal-block
// substitutions into 16×16 matrix-vector products.
// ------------------------------------------------------------------------
template <class LT = KLayout>
__device__ __forceinline__ void invert_diag_block(float* __restrict__ K, const LT& L, int b,
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
// Signed Cholesky of the packed matrix K (layout L), right-looking, 16-wide
// panels:
//   for each block b:
//     (1) panel factorisation by the whole CTA: every thread owns one (or
//         RPT) rows of the panel [k0, N4) × [k0, k0+16) in registers; per
//         column k one barrier, then every thread reads the pivot and the
//         column-k entries of the diagonal-block rows (broadcast), scales its
//         own l_ik and updates its row; diagonal-block rows publish their next
//         column entry for the next step.
//     (2) rank-16 update of the trailing lower triangle (SYRK): 32×32
//         super-tiles, one warp each, 8×4 strided register tiles.
//   finally every warp inverts diagonal blocks (W_b = L_bb⁻¹, for solve_qd).
// A pivot on the wrong side of ±θ is replaced by ±θ (reading Q12) and
// counted.  On exit K holds L (M = L S Lᵀ) and rinv[k] = 1/L[k][k].
// ------------------------------------------------------------------------
template <int NT, bool TAB = false, int MAXN4 = 256>
__device__ int factor_qd(float* __restrict__ K, const KLayout& L, const float theta, float* __restrict__ rinv,
                         int* __restrict__ flag, float* __restrict__ colT, const int* __restrict__ tab = nullptr) {
  constexpr int NW = NT / 32;
  constexpr int RPT = (MAXN4 + NT - 1) / NT;  // rows per thread (N4 ≤ MAXN4)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N4 = L.N4, npos = L.npos;
  int nfloor = 0;
  long long tc0 = clock64(), tpan = 0, tsyrk = 0;
  for (int b = 0; b < L.NB; ++b) {
    const int k0 = KB * b, kb = L.bw(b), k1 = k0 + kb;
    const float* D = K + L.off(k0) + k0;  // diagonal block, row j at D + j*Lb
    const int Lb = L.len(b);
    // ---- (1) panel factorisation, unscaled LDLᵀ updates a_ij −= a_ik a_jk / a_kk:
    //      column k is read-only during step k, so one barrier per column
    //      suffices.  Each thread keeps its row's remaining panel columns in a
    //      register window that shifts by one per step (w[0] = column k), and
    //      stores l_ik = a_ik s_k / l_kk as soon as column k is final. ----------
    //      The current column k of the diagonal-block rows is published in
    //      colT[k][·] at positions RELATIVE to k (colT[k][j] = a_{k+j,k}), so
    //      every thread reads it as four float4 broadcasts at static offsets,
    //      matching its shifting window.  Warps whose rows all lie past N4 skip
    //      the step (barriers only).
    float w[RPT][KB];
    float* rowp[RPT];
    bool has[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int i = k0 + tid + u * NT;
      has[u] = i < N4;
      rowp[u] = K + row_off<TAB>(L, tab, has[u] ? i : k0) + k0;
#pragma unroll
      for (int j4 = 0; j4 < KB / 4; ++j4) {
        const float4 t = (has[u] && 4 * j4 < kb) ? reinterpret_cast<const float4*>(rowp[u])[j4]
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        w[u][4 * j4] = t.x; w[u][4 * j4 + 1] = t.y; w[u][4 * j4 + 2] = t.z; w[u][4 * j4 + 3] = t.w;
      }
    }
    // columns 0..PC-1 as loaded (NT ≥ 16: the diagonal-block rows have u = 0)
    if (tid < KB) {
#pragma unroll
      for (int q = 0; q < PC; ++q)
        if (tid >= q) colT[KB * q + tid - q] = tid < kb ? w[0][q] : 0.f;
    }
    // warp-uniform: does any row of (warp, u) lie inside the panel?
    bool wact[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) wact[u] = k0 + 32 * warp + u * NT < N4;
    // PC columns per barrier (kb is a multiple of 4).  Published per step:
    // columns k..k+PC-1 updated through column k−1; every thread brings them
    // up to date itself (a PC×16 triangle of redundant FMAs, with exactly the
    // rounding the owners of those rows apply to their own entries) instead of
    // waiting for more barriers.  The panel reads columns only from colT, so
    // the l values go to K at once.
    for (int k = 0; k < kb; k += PC) {
      __syncthreads();
      if (!wact[0]) continue;  // rows of u ≥ 1 lie further down: inactive too
      float c[PC][KB];  // c[q][j] = a_{k+q+j, k+q}
#pragma unroll
      for (int q = 0; q < PC; ++q) {
        const float4* pq = reinterpret_cast<const float4*>(colT + KB * (k + q));
#pragma unroll
        for (int j4 = 0; j4 < KB / 4; ++j4) {
          const float4 t = pq[j4];
          c[q][4 * j4] = t.x; c[q][4 * j4 + 1] = t.y; c[q][4 * j4 + 2] = t.z; c[q][4 * j4 + 3] = t.w;
        }
      }
      float dq[PC], rsq[PC], inv[PC], sr[PC];
      int nf = 0;
#pragma unroll
      for (int q = 0; q < PC; ++q) {
#pragma unroll
        for (int r = 0; r < q; ++r)
#pragma unroll
          for (int j = 0; j + q - r < KB; ++j) c[q][j] = fmaf(-c[r][q - r + j] * inv[r], c[r][q - r], c[q][j]);
        const float sg = sgn_of(k0 + k + q, npos);
        float d = sg * c[q][0];
        const bool fl = !(d >= theta);
        if (fl) d = theta;
        nf += fl;
        const float rs = rsqrtf(d);
        dq[q] = d; rsq[q] = rs; inv[q] = sg * rs * rs; sr[q] = sg * rs;
      }
      if (tid == 0) {
#pragma unroll
        for (int q = 0; q < PC; ++q) rinv[k0 + k + q] = rsq[q];
        nfloor += nf;
      }
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        if (!wact[u]) continue;
        const int il = tid + u * NT;  // row index relative to k0
        if (has[u] && il >= k) {
          bool live = true;
#pragma unroll
          for (int q = 0; q < PC; ++q) {
            if (live) {
              if (il == k + q) {
                rowp[u][k + q] = dq[q] * rsq[q];  // l_kk
                live = false;
              } else {
                const float f = -w[u][q] * inv[q];
                rowp[u][k + q] = w[u][q] * sr[q];
#pragma unroll
                for (int j = q + 1; j < KB; ++j) w[u][j] = fmaf(f, c[q][j - q], w[u][j]);
              }
            }
          }
          if (live && u == 0 && il < kb) {  // publish columns k+PC.. (updated through k+PC−1)
#pragma unroll
            for (int t = 0; t < PC; ++t)
              if (il >= k + PC + t) colT[KB * (k + PC + t) + il - k - PC - t] = w[u][PC + t];
          }
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) w[u][j] = j + PC < KB ? w[u][j + PC] : 0.f;
      }
    }
    __syncthreads();
    { const long long t = clock64(); tpan += t - tc0; tc0 = t; }
    // ---- (2) trailing update A22 −= L21 S_b L21ᵀ --------------------------------
    //      32-row × 16-column tiles of the lower triangle, one warp each
    //      (8×2 strided register tile per lane): twice as many tiles as 32×32
    //      ones, so the 4 warps stay balanced on the small trailing matrices
    //      of path 1 (T = 3 row blocks: 12 tiles instead of 6).
    if (k1 < N4) {
      const int Tn = N4 - k1;
      const int T = (Tn + 31) >> 5, T16 = (Tn + 15) >> 4;
      const int nst = T * (T + 1) - (2 * T - T16);  // Σ_I min(2I + 2, T16)
      const int ty = lane >> 3, tx = lane & 7;
      for (int st = warp; st < nst; st += NW) {
        int I = 0, J = st;
        while (J >= min(2 * I + 2, T16)) { J -= min(2 * I + 2, T16); ++I; }
        const int rb = k1 + 32 * I + ty, cb = k1 + 16 * J + tx;
        int roff[8], coff[2];
        bool rok[8], cok[2];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = rb + 4 * q;
          rok[q] = r < N4;
          roff[q] = rok[q] ? row_off<TAB>(L, tab, r) : 0;
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int cc = cb + 8 * c;
          cok[c] = cc < N4;
          coff[c] = cok[c] ? row_off<TAB>(L, tab, cc) : 0;
        }
        float acc[8][2];
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            acc[q][c] = (rok[q] && cok[c] && cb + 8 * c <= rb + 4 * q) ? K[roff[q] + cb + 8 * c] : 0.f;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          // S_b applied to the column operand (npos is a multiple of 4)
          const float sq = k0 + 4 * q4 < npos ? -1.f : 1.f;
          float4 lc[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            float4 t = cok[c] ? *reinterpret_cast<const float4*>(K + coff[c] + k0 + 4 * q4)
                              : make_float4(0, 0, 0, 0);
            t.x *= sq; t.y *= sq; t.z *= sq; t.w *= sq;
            lc[c] = t;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 lr = rok[q] ? *reinterpret_cast<const float4*>(K + roff[q] + k0 + 4 * q4)
                                     : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              float t = acc[q][c];
              t = fmaf(lr.x, lc[c].x, t);
              t = fmaf(lr.y, lc[c].y, t);
              t = fmaf(lr.z, lc[c].z, t);
              t = fmaf(lr.w, lc[c].w, t);
              acc[q][c] = t;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int cc = cb + 8 * c;
            // lower triangle only (a diagonal block's upper part is never touched)
            if (rok[q] && cok[c] && cc <= rb + 4 * q) K[roff[q] + cc] = acc[q][c];
          }
      }
      __syncthreads();
    }
    { const long long t = clock64(); tsyrk += t - tc0; tc0 = t; }
  }
  // ---- W_b = L_bb⁻¹ for every diagonal block (solve_qd) -------------------------
  for (int b = warp; b < L.NB; b += NW) invert_diag_block(K, L, b, rinv);
  if (tid == 0) *flag = nfloor;
  __syncthreads();
  if (tid == 0 && g_fac_on) {
    atomicAdd(&g_fac_cycles[0], (unsigned long long)tpan);
    atomicAdd(&g_fac_cycles[1], (unsigned long long)tsyrk);
    atomicAdd(&g_fac_cycles[2], (unsigned long long)(clock64() - tc0));
    atomicAdd(&g_fac_cycles[3], 1ull);
  }
  const int r = *flag;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------------
// Large-N variant (path 2): K lives in a per-CTA GLOBAL workspace (L2
// resident for config 4), the panel rows are streamed instead of held in
// registers.  Per 16-wide block:
//   (a) warp 0 factors the diagonal block (unscaled LDLᵀ updates, register
//       window per lane, column broadcast through a 16-float smem scratch),
//       writes L_bb to K and to the smem scratch `l11` (16×16);
//   (b) every thread solves rows of the panel below (x L_bbᵀ = a, l = S x),
//       L_bb read from smem (broadcast);
//   (c) rank-16 update of the trailing lower triangle (32×32 super-tiles per
//       warp, as in factor_qd).
// Then the diagonal-block inverses W_b.  scr: ≥ 16·17 + 16 floats of smem.
// ------------------------------------------------------------------------
// Columns [c0, c1) of the factorisation (c0 a multiple of 16, c1 a multiple
// of 16 or N4): the 16-wide blocks of the range are factored together with
// every row below them, and the trailing update touches only columns < c1
// (factor_tc's tensor-core left-looking update brings later columns up to
// date).  Returns the number of floored pivots (thread 0's count).
// A column panel [c0, c0 + S') of the packed matrix copied to a dense
// shared-memory array: row i (≥ c0) at (i − c0)·S, column j at j − c0 (the
// caller offsets the base pointer by −c0).  Same interface as KLayout for
// factor_big_range.
struct PanelLayout {
  int N4, NB, npos, c0, S;
  KLayout base;
  __device__ __forceinline__ int off(int i) const { return (i - c0) * S; }
  __device__ __forceinline__ int len(int) const { return S; }
  __device__ __forceinline__ int bw(int b) const { return base.bw(b); }
};

// QS: rows of a 32×32 super-tile a lane accumulates per pass (8: one pass;
// 4: two passes with half the accumulator registers)
template <int NT, class LT = KLayout, int QS = 8>
__device__ int factor_big_range(float* __restrict__ K, const LT& L, const float theta, float* __restrict__ rinv,
                                float* __restrict__ scr, const int c0, const int c1) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N4 = L.N4, npos = L.npos;
  float* l11 = scr;            // [16][17]
  float* colb = scr + 16 * 17;  // [16] column broadcast
  int nfloor = 0;
  for (int b = c0 / KB; b < L.NB && KB * b < c1; ++b) {
    const int k0 = KB * b, kb = L.bw(b), k1 = k0 + kb;
    const int Lb = L.len(b);
    // ---- (a) diagonal block ---------------------------------------------------------
    if (warp == 0) {
      const int r = lane;
      float* rowr = K + L.off(k0 + (r < kb ? r : 0)) + k0;
      float w[KB];
#pragma unroll
      for (int j = 0; j < KB; ++j) w[j] = (r < kb && j < kb) ? rowr[j] : 0.f;
      for (int k = 0; k < kb; ++k) {
        if (r < kb) colb[r] = w[0];  // current column-k entry of row r
        __syncwarp();
        const float s = sgn_of(k0 + k, npos);
        float d = s * colb[k];
        const bool fl = !(d >= theta);
        if (fl) d = theta;
        const float rs = rsqrtf(d);
        const float inv = s * rs * rs;
        float col[KB];
#pragma unroll
        for (int j = 1; j < KB; ++j) col[j] = colb[min(k + j, KB - 1)];
        __syncwarp();
        if (lane == 0) { rinv[k0 + k] = rs; nfloor += fl; }
        if (r < kb && r >= k) {
          float lv;
          if (r == k) {
            lv = d * rs;
          } else {
            const float f = -w[0] * inv;
            lv = w[0] * s * rs;
#pragma unroll
            for (int j = 1; j < KB; ++j) w[j] = fmaf(f, col[j], w[j]);
          }
          rowr[k] = lv;
          l11[r * 17 + k] = lv;
        }
#pragma unroll
        for (int j = 0; j + 1 < KB; ++j) w[j] = w[j + 1];
        w[KB - 1] = 0.f;
      }
    }
    __syncthreads();
    if (k1 >= N4) break;
    // ---- (b) TRSM of the panel rows below ---------------------------------------------
    for (int i = k1 + tid; i < N4; i += NT) {
      float* row = K + L.off(i) + k0;
      float a[KB];
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float4 t = reinterpret_cast<const float4*>(row)[j4];
        a[4 * j4] = t.x; a[4 * j4 + 1] = t.y; a[4 * j4 + 2] = t.z; a[4 * j4 + 3] = t.w;
      }
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const float xk = a[k] * rinv[k0 + k];
        a[k] = xk;
#pragma unroll
        for (int j = k + 1; j < KB; ++j) a[j] = fmaf(-xk, l11[j * 17 + k], a[j]);
      }
#pragma unroll
      for (int j4 = 0; j4 < 4; ++j4) {
        const float s0 = sgn_of(k0 + 4 * j4, npos);
        reinterpret_cast<float4*>(row)[j4] =
            make_float4(s0 * a[4 * j4], s0 * a[4 * j4 + 1], s0 * a[4 * j4 + 2], s0 * a[4 * j4 + 3]);
      }
    }
    __syncthreads();
    // ---- (c) trailing update A22 −= L21 S_b L21ᵀ, columns < c1 ---------------------------
    if (k1 < c1) {
      const int T = (N4 - k1 + 31) >> 5;      // 32-row tiles below
      const int JT = (c1 - k1 + 31) >> 5;     // 32-column tiles inside the range
      const int ncol = c1 < N4 ? c1 : N4;     // column bound of this update
      const int nst = JT * T - JT * (JT - 1) / 2;  // tiles (I, J): J < JT, J ≤ I < T
      const int ty = lane >> 3, tx = lane & 7;
      for (int st = warp; st < nst; st += NW) {
        int J = 0, rem = st;
        while (rem >= T - J) { rem -= T - J; ++J; }
        const int I = J + rem;
        const int cb = k1 + 32 * J + tx;
        int coff[4];
        bool cok[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int cc = cb + 8 * c;
          cok[c] = cc < ncol;
          coff[c] = cok[c] ? L.off(cc) : 0;
        }
#pragma unroll 1
        for (int hh = 0; hh < 8 / QS; ++hh) {
        const int rb = k1 + 32 * I + ty + 4 * QS * hh;
        int roff[QS];
        bool rok[QS];
#pragma unroll
        for (int q = 0; q < QS; ++q) {
          const int rr = rb + 4 * q;
          rok[q] = rr < N4;
          roff[q] = rok[q] ? L.off(rr) : 0;
        }
        float acc[QS][4];
#pragma unroll
        for (int q = 0; q < QS; ++q)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            acc[q][c] = (rok[q] && cok[c] && cb + 8 * c <= rb + 4 * q) ? K[roff[q] + cb + 8 * c] : 0.f;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float sq = k0 + 4 * q4 < npos ? -1.f : 1.f;
          float4 lc[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float4 t = cok[c] ? *reinterpret_cast<const float4*>(K + coff[c] + k0 + 4 * q4)
                              : make_float4(0, 0, 0, 0);
            t.x *= sq; t.y *= sq; t.z *= sq; t.w *= sq;
            lc[c] = t;
          }
#pragma unroll
          for (int q = 0; q < QS; ++q) {
            const float4 lr = rok[q] ? *reinterpret_cast<const float4*>(K + roff[q] + k0 + 4 * q4)
                                     : make_float4(0, 0, 0, 0);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float t = acc[q][c];
              t = fmaf(lr.x, lc[c].x, t);
              t = fmaf(lr.y, lc[c].y, t);
              t = fmaf(lr.z, lc[c].z, t);
              t = fmaf(lr.w, lc[c].w, t);
              acc[q][c] = t;
            }
          }
        }
#pragma unroll
        for (int q = 0; q < QS; ++q)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int cc = cb + 8 * c;
            if (rok[q] && cok[c] && cc <= rb + 4 * q) K[roff[q] + cc] = acc[q][c];
          }
        }
      }
    }
    __syncthreads();
  }
  return nfloor;
}

template <int NT>
__device__ int factor_big(float* __restrict__ K, const KLayout& L, const float theta, float* __restrict__ rinv,
                          int* __restrict__ flag, float* __restrict__ scr) {
  const int nfloor = factor_big_range<NT>(K, L, theta, rinv, scr, 0, L.N4);
  for (int b = threadIdx.x >> 5; b < L.NB; b += NT / 32) invert_diag_block(K, L, b, rinv);
  if (threadIdx.x == 0) *flag = nfloor;
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
template <int NT, bool TAB = false, bool UNR = false>
__device__ void solve_qd(const float* __restrict__ K, const KLayout& L, const float* __restrict__ rinv,
                         float* __restrict__ rhs, const int* __restrict__ tab = nullptr, bool fwd = true) {
  const int tid = threadIdx.x;
  const int N4 = L.N4;
  // forward: L u = b (fwd = false: already done during the factorisation, rhs holds u)
  for (int b = 0; fwd && b < L.NB; ++b) {
    const int k0 = KB * b, kb = L.bw(b);
    const float* D = K + row_off<TAB>(L, tab, k0) + k0;
    const int Lb = L.len(b);
    if (tid < 32) {
      const int t = tid;
      float r[KB];
#pragma unroll
      for (int c = 0; c < KB; ++c) r[c] = c < kb ? rhs[k0 + c] : 0.f;
      const float rt = t < kb ? rhs[k0 + t] : 0.f;  // r[t] without dynamic register indexing
      __syncwarp();
      if (t < kb) {
        float acc = rinv[k0 + t] * rt;
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
        const float4* row = reinterpret_cast<const float4*>(K + row_off<TAB>(L, tab, i) + k0);
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
    const float* D = K + row_off<TAB>(L, tab, k0) + k0;
    const int Lb = L.len(b);
    if (tid < 32) {
      const int t = tid;
      float r[KB];
#pragma unroll
      for (int c = 0; c < KB; ++c) r[c] = c < kb ? rhs[k0 + c] : 0.f;
      const float rt = t < kb ? rhs[k0 + t] : 0.f;  // r[t] without dynamic register indexing
      __syncwarp();
      if (t < kb) {
        float acc = rinv[k0 + t] * rt;
        const float* Dt = D + t * Lb;  // W[r][t] for r > t lives in row t, column r
#pragma unroll
        for (int c = 0; c < KB; ++c)
          if (c > t && c < kb) acc = fmaf(Dt[c], r[c], acc);
        rhs[k0 + t] = acc;
      }
    }
    __syncthreads();
    if (b > 0) {
      const float* Bk = K + row_off<TAB>(L, tab, k0);
      if constexpr (UNR) {  // (K in global memory) L2 prefetch of the next block row, one per 128-byte line
        const int kp = k0 - KB, nl = (kp + 31) >> 5;
        const float* Bp = K + row_off<TAB>(L, tab, kp);
        const int Lp = L.len(b - 1);
        for (int q = tid; q < KB * nl; q += NT) {
          const int i = q / nl, c = (q - i * nl) << 5;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(Bp + i * Lp + c));
        }
      }
      for (int j = tid; j < k0; j += NT) {
        float acc = rhs[j];
        if constexpr (UNR) {
          // (batched engine, K in global memory) all 16 loads in flight
          float lv[KB];
#pragma unroll
          for (int i = 0; i < KB; ++i) lv[i] = i < kb ? Bk[i * Lb + j] : 0.f;
#pragma unroll
          for (int i = 0; i < KB; ++i) acc = fmaf(-lv[i], i < kb ? rhs[k0 + i] : 0.f, acc);
        } else {
          for (int i = 0; i < kb; ++i) acc = fmaf(-Bk[i * Lb + j], rhs[k0 + i], acc);
        }
        rhs[j] = acc;
      }
      __syncthreads();
    }
  }
}

}  // namespace qpb

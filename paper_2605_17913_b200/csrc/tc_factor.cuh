// tc_factor.cuh — large-N factorisation with the Schur-complement updates on
// the 5th-generation tensor cores ("the tiled Schur
// update"; the factorisation is the dominant cost).
//
// Left-looking by panels of w = 64 columns.  For each
// panel [c0, c0+w):
//   (1) bring it up to date with every earlier column in one GEMM per
//       128-row tile:  K[i][c0+c] −= Σ_{k<c0} L[i][k]·S_k·L[c0+c][k], the sum
//       accumulated in TMEM by tcgen05.mma.kind::tf32 (3×TF32 split, K-major
//       operands staged from the packed rows, which are contiguous in k), the
//       subtraction done in a coalesced epilogue;
//   (2) factor the panel with factor_big_range (16-wide blocks: warp-factored
//       diagonal block, TRSM of the rows below, FP32 trailing update confined
//       to the panel's columns) — on a dense copy of the panel in the shared-
//       memory KKT buffer when K lives in the global workspace and the panel
//       fits, else in place.
// The operand loads of both loops are backed by L2 prefetches three K chunks
// ahead (config 5's workspace, 19 MB per CTA, does not stay in L2).
// Traffic: each panel's update reads the rows [i][0:c0] once (≈ N³/(6w)
// floats in total) instead of the right-looking read-modify-write of the
// whole trailing matrix per 16 columns (≈ N³/24 floats).
#pragma once
#include "ipm_cta.cuh"
#include "tc_syrk.cuh"

namespace qpb {

__device__ int g_tc_w;  // panel width override (QPB200_TC_W experiments; 0 = default)
__device__ unsigned long long g_tcf_cycles[4];  // diagnostics: tensor-core updates, panels, inverses, count

// kind::tf32 instruction descriptor for M = 128, N = nn (multiple of 16, ≤ 256)
__device__ __forceinline__ uint32_t tc_idesc_n(int nn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(nn >> 3) << 17) | ((uint32_t)(tc::TM >> 4) << 24);
}

// Rows [i0, i0+128) of panel [c0, c0+w) (w ≤ 128, multiple of 16; c0 > 0).
template <int NT>
__device__ void tc_left_update(const tc::TcState& s, float* __restrict__ K, const KLayout& L, const int c0, const int w,
                               const int i0) {
  using namespace tc;
  constexpr int UA = (TK / 4) * TM / NT;   // A units (one row, 4 consecutive k) per thread
  constexpr int UB = (TK / 4) * 128 / NT;  // B units per thread (w ≤ 128)
  constexpr int PF = 3;                     // L2 prefetch distance in K chunks
  const int tid = threadIdx.x;
  const int N4 = L.N4, npos = L.npos;
  const uint32_t tmem = *s.tmem_slot;
  uint32_t phase = *s.phase_slot;
  const uint32_t idesc = tc_idesc_n(w);
  float4 ra[UA], rb[UB];
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int unit = tid + u * NT, kc = unit / TM, m = unit - kc * TM;
      const int i = i0 + m, k = k0 + 4 * kc;
      ra[u] = (i < N4 && k < c0) ? *reinterpret_cast<const float4*>(K + L.off(i) + k) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int unit = tid + u * NT, kc = unit / w, c = unit - kc * w;
      const int j = c0 + c, k = k0 + 4 * kc;
      rb[u] = (kc < TK / 4 && j < N4 && k < c0) ? *reinterpret_cast<const float4*>(K + L.off(j) + k)
                                                : make_float4(0, 0, 0, 0);
    }
  };
  // the operand rows of chunk k0 into L2 (the workspace of a large system does
  // not stay L2-resident: config 5's is 19 MB per CTA)
  auto prefetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int unit = tid + u * NT, kc = unit / TM, m = unit - kc * TM;
      const int i = i0 + m, k = k0 + 4 * kc;
      if (i < N4 && k < c0 && (k & 31) == 0)  // one prefetch per 128-B row segment
        asm volatile("prefetch.global.L2 [%0];" ::"l"(K + L.off(i) + k));
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int unit = tid + u * NT, kc = unit / w, c = unit - kc * w;
      const int j = c0 + c, k = k0 + 4 * kc;
      if (kc < TK / 4 && j < N4 && k < c0 && (k & 31) == 0)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(K + L.off(j) + k));
    }
  };
  auto split = [](float4 v, float4& hi, float4& lo) {
    hi.x = to_tf32(v.x); lo.x = to_tf32(v.x - hi.x);
    hi.y = to_tf32(v.y); lo.y = to_tf32(v.y - hi.y);
    hi.z = to_tf32(v.z); lo.z = to_tf32(v.z - hi.z);
    hi.w = to_tf32(v.w); lo.w = to_tf32(v.w - hi.w);
  };
  auto store = [&](int k0) {
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const int unit = tid + u * NT, kc = unit / TM, m = unit - kc * TM;
      float4 hi, lo;
      split(ra[u], hi, lo);
      const int o = op_offset(m, 4 * kc);
      *reinterpret_cast<float4*>(s.ahi + o) = hi;
      *reinterpret_cast<float4*>(s.alo + o) = lo;
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int unit = tid + u * NT, kc = unit / w, c = unit - kc * w;
      if (kc < TK / 4) {
        float4 v = rb[u];
        if (k0 + 4 * kc >= npos) { v.x = -v.x; v.y = -v.y; v.z = -v.z; v.w = -v.w; }  // S_k (npos % 4 == 0)
        float4 hi, lo;
        split(v, hi, lo);
        const int o = op_offset(c, 4 * kc);
        *reinterpret_cast<float4*>(s.bhi + o) = hi;
        *reinterpret_cast<float4*>(s.blo + o) = lo;
      }
    }
  };
  load(0);
  for (int k0 = 0; k0 < c0; k0 += TK) {
    store(k0);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ahi = smem_u32(s.ahi), alo = smem_u32(s.alo), bhi = smem_u32(s.bhi), blo = smem_u32(s.blo);
#pragma unroll
      for (int ks = 0; ks < TK / 8; ++ks) {
        const uint32_t off = ks * 2 * 128;  // bytes per MMA k-step of 8 (two K chunks)
        const uint32_t acc0 = (k0 > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, make_desc(ahi + off), make_desc(bhi + off), idesc, acc0);
        mma_tf32(tmem, make_desc(ahi + off), make_desc(blo + off), idesc, 1u);
        mma_tf32(tmem, make_desc(alo + off), make_desc(bhi + off), idesc, 1u);
      }
      commit(s.mbar);
    }
    if (k0 + TK < c0) load(k0 + TK);  // overlaps the MMAs of this chunk
    if (k0 + PF * TK < c0) prefetch(k0 + PF * TK);  // L2 prefetch PF chunks ahead (no registers held)
    mbar_wait(s.mbar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  if (tid == 0) *s.phase_slot = phase;
  // epilogue: K[i][c0+c] −= acc (lower triangle), coalesced row segments
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int NH = NT / 128;
  const int q = warp & 3, half = warp >> 2;
  float* T = s.ahi + warp * (32 * 33);
#pragma unroll 1
  for (int cc = 32 * half; cc < w; cc += 32 * NH) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)cc, v);
#pragma unroll
    for (int c = 0; c < 32; ++c) T[lane * 33 + c] = v[c];
    __syncwarp();
    const int c = cc + lane, j = c0 + c;
    float kv[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int i = i0 + 32 * q + r;
      kv[r] = (c < w && i < N4 && j <= i) ? K[L.off(i) + j] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int i = i0 + 32 * q + r;
      if (c < w && i < N4 && j <= i) K[L.off(i) + j] = kv[r] - T[r * 33 + lane];
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
}

// Signed Cholesky M = L S Lᵀ of the packed matrix K (layout L) for large N;
// same output contract as factor_qd / factor_big.
template <int NT>
__device__ int factor_tc(float* __restrict__ K, const KLayout& L, const float theta, float* __restrict__ rinv,
                         int* __restrict__ flag, float* __restrict__ scr, const tc::TcState& ts,
                         float* __restrict__ pbuf = nullptr, int pcap = 0) {
  const int N4 = L.N4;
  const int w = g_tc_w > 0 ? g_tc_w : 64;  // measured: config 4 best at 64 (16: -20 %, 32: -5 %), config 5 flat for 64-128
  int nfloor = 0;
  long long t0 = clock64(), tup = 0, tpan = 0;
  for (int c0 = 0; c0 < N4; c0 += w) {
    const int c1 = c0 + w < N4 ? c0 + w : N4;
    if (c0 > 0) {
      const int wn = (c1 - c0 + 15) & ~15;  // MMA N (columns ≥ N4 are zero)
      for (int i0 = c0; i0 < N4; i0 += tc::TM) tc_left_update<NT>(ts, K, L, c0, wn, i0);
    }
    { const long long t = clock64(); tup += t - t0; t0 = t; }
    // the panel's rows [c0, N4) × columns [c0, c1) are factored in shared
    // memory when they fit the (otherwise idle: K lives in the global
    // workspace) smem KKT buffer `pbuf`; else in place in global memory
    constexpr int PS = 68;  // panel row stride: 64 columns + 4 (rows 16-B aligned, odd multiple of 16 B)
    if (pbuf && c1 - c0 <= 64 && (N4 - c0) * PS <= pcap) {
      const int nr = N4 - c0, wc = c1 - c0;
      for (int e = threadIdx.x; e < nr * (wc >> 2); e += NT) {
        const int r = e / (wc >> 2), q = e - r * (wc >> 2);
        const int i = c0 + r, j = c0 + 4 * q;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j <= i) v = *reinterpret_cast<const float4*>(K + L.off(i) + j);  // (j ≤ i: within row i)
        *reinterpret_cast<float4*>(pbuf + r * PS + 4 * q) = v;
      }
      __syncthreads();
      PanelLayout P;
      P.N4 = L.N4; P.NB = L.NB; P.npos = L.npos; P.c0 = c0; P.S = PS; P.base = L;
      nfloor += factor_big_range<NT>(pbuf - c0, P, theta, rinv, scr, c0, c1);
      for (int e = threadIdx.x; e < nr * (wc >> 2); e += NT) {
        const int r = e / (wc >> 2), q = e - r * (wc >> 2);
        const int i = c0 + r, j = c0 + 4 * q;
        if (j <= i) *reinterpret_cast<float4*>(K + L.off(i) + j) = *reinterpret_cast<const float4*>(pbuf + r * PS + 4 * q);
      }
      __syncthreads();
    } else {
      nfloor += factor_big_range<NT>(K, L, theta, rinv, scr, c0, c1);
    }
    { const long long t = clock64(); tpan += t - t0; t0 = t; }
  }
  for (int b = threadIdx.x >> 5; b < L.NB; b += NT / 32) invert_diag_block(K, L, b, rinv);
  if (threadIdx.x == 0 && g_fac_on) {  // diagnostics (QPB200_PHASE_PROFILE)
    atomicAdd(&g_tcf_cycles[0], (unsigned long long)tup);
    atomicAdd(&g_tcf_cycles[1], (unsigned long long)tpan);
    atomicAdd(&g_tcf_cycles[2], (unsigned long long)(clock64() - t0));
    atomicAdd(&g_tcf_cycles[3], 1ull);
  }
  if (threadIdx.x == 0) *flag = nfloor;
  __syncthreads();
  const int r = *flag;
  __syncthreads();
  return r;
}

}  // namespace qpb

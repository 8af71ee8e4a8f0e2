// kr_gemm.cuh — KKT assembly for a batch whose G is SHARED (stride 0; the
// end-to-end-learning setting of BASELINE config 4) as ONE dense
// tensor-core GEMM over the batch, fed by the TMA bulk-copy engine.
//
// Row i ≥ j of problem b's (1,1) block is (the bounded scaling)
//     H_b[i][j] = Q[i][j] + Σ_k ω_b[k] G[k][i] G[k][j].
// With the pair index t = i(i+1)/2 + j over the lower triangle (including
// the identity padding rows n..n4) and GG[k][t] = G[k][i] G[k][j] (the
// Khatri-Rao square of G, fixed for the whole call), the whole batch is
//     Hvec = Ω · GGᵀ      Ω: [active problems × p],  GG: [p × n4(n4+1)/2]
// — M = problems, N = pairs, K = constraints: a plain GEMM with no wasted
// tile area (a per-problem 128×128 SYRK tiling of n = 200 computes 2.4× the
// triangle) and with both operands read straight from L2 by bulk copies.
//
// Accuracy: 3×TF32 split (x = x_hi + x_lo, hi = tf32(x), lo = tf32(x − hi);
// D = Ω_hi·GG_hiᵀ + Ω_hi·GG_loᵀ + Ω_lo·GG_hiᵀ) keeps f32-level accuracy.
//
// Operand storage: both operands are stored in global memory ALREADY in the
// canonical no-swizzle K-major UMMA tile layout (tc_syrk.cuh op_offset), one
// contiguous 16 KB (Ω: 128 rows × 32 k) or 32 KB (GG: 256 pairs × 32 k) block
// per (tile, K chunk), hi and lo separately, so each stage of the pipeline is
// four `cp.async.bulk` copies (SASS UBLKCP) completing on an mbarrier
// (expect_tx).  Ω rows are written by bnd_resid / bnd_begin for the problem's
// slot in this iteration's list of iterating problems; GG by kr_prep once per
// call.
//
// Kernel: persistent, one CTA per SM, 192 threads, (128 problems × 256
// pairs) output tiles, 2-stage ring of 96 KB: a producer warp issues the bulk
// copies, an MMA warp issues tcgen05.mma.cta_group::1.kind::tf32 (M = 128,
// N = 256, K = 8) into one of two TMEM accumulators (2 × 256 fp32 columns)
// and commits each stage back to the producer, and four epilogue warps drain
// the other accumulator (tcgen05.ld.32x32b.x32), transpose through shared
// memory and write each problem's pairs into its packed KKT workspace
// (ipm_cta.cuh layout), adding Q and the padding identity, and record
// max|diag| (the pivot floor's scale) per problem — the epilogue of one tile
// overlapping the copies and MMAs of the next.
#pragma once
#include "ipm_cta.cuh"
#include "tc_syrk.cuh"

namespace qpb {
namespace kr {

constexpr int BM = 128, BN = 256, BK = 32;
constexpr int A_FL = BM * BK, B_FL = BN * BK;               // floats per tile chunk
constexpr int STAGE_FL = 2 * A_FL + 2 * B_FL;               // Ω hi, lo; GG hi, lo
constexpr int STAGES = 2;
constexpr int SMEM_BYTES = STAGES * STAGE_FL * 4 + 256;     // + barriers, TMEM slot

__host__ __device__ inline int nkc(int p) { return (p + BK - 1) / BK; }
__host__ __device__ inline int npairs(int n4) { return n4 * (n4 + 1) / 2; }

// element (row r, constraint k) of the operand whose tiles hold R rows
template <int R>
__device__ __forceinline__ long long at(int row, int k, int nk) {
  const int t = row / R, r = row - t * R, kc = k / BK, kk = k - kc * BK;
  return ((long long)t * nk + kc) * (R * BK) + ((r >> 3) * (BK / 4) + (kk >> 2)) * 32 + (r & 7) * 4 + (kk & 3);
}

__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = tc::to_tf32(x);
  lo = tc::to_tf32(x - hi);
}

// Ω row of `slot` (ω_k for k < p, zero up to the padded K).
template <int NT>
__device__ __forceinline__ void write_omega(float* whi, float* wlo, int slot, const float* om, int p, bool ones) {
  const int nk = nkc(p);
  for (int k = threadIdx.x; k < nk * BK; k += NT) {
    const float w = k < p ? (ones ? 1.f : om[k]) : 0.f;
    float hi, lo;
    split(w, hi, lo);
    const long long o = at<BM>(slot, k, nk);
    whi[o] = hi;
    wlo[o] = lo;
  }
}

// GG[k][t] = G[k][i] G[k][j] for the pair t = (i, j), zero past n / p.
__global__ void __launch_bounds__(256) kr_prep(const float* __restrict__ G, int n, int n4, int p, float* gghi,
                                               float* gglo) {
  const int nk = nkc(p), np = npairs(n4);
  const int ntile = (np + BN - 1) / BN;
  const long long tot = (long long)ntile * BN * nk * BK;
  for (long long e = blockIdx.x * 256ll + threadIdx.x; e < tot; e += (long long)gridDim.x * 256) {
    const int t = (int)(e / (nk * BK)), k = (int)(e - (long long)t * nk * BK);
    float v = 0.f;
    if (t < np && k < p) {
      int i = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
      while ((i + 1) * (i + 2) / 2 <= t) ++i;
      while (i * (i + 1) / 2 > t) --i;
      const int j = t - i * (i + 1) / 2;
      if (i < n && j < n) v = __ldg(G + (size_t)k * n + i) * __ldg(G + (size_t)k * n + j);
    }
    float hi, lo;
    split(v, hi, lo);
    const long long o = at<BN>(t, k, nk);
    gghi[o] = hi;
    gglo[o] = lo;
  }
}

struct GemmArgs {
  const float *whi, *wlo, *gghi, *gglo;
  const int* count;    // iterating problems (slots 0..count-1)
  const int* slotmap;  // slot -> problem (chunk-local index)
  float* kw;           // KKT workspaces [B][kstride]
  long long kstride;
  float* st;           // state blocks (BScal header: pa, dmax)
  long long st_stride;
  const float* Q;
  long long sQ;
  int n, n4, m, p;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(mbar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc::smem_u32(mbar))
               : "memory");
}

// kind::tf32, M = 128, N = 256, both K-major
__device__ __forceinline__ uint32_t idesc_256() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// Persistent, warp-specialised: grid = min(tiles, SMs), tiles (problem tile
// fastest) strided over the CTAs.  Warp 4 produces (bulk copies into the
// 2-stage ring), warp 5 issues the MMAs into one of TWO TMEM accumulators
// (2 × 256 columns), warps 0-3 drain the other accumulator (epilogue) at the
// same time — so the epilogue of tile t overlaps the loads and MMAs of tile
// t + 1.  mbarriers: full/empty per ring stage, tfull/tempty per accumulator.
constexpr int WS_THREADS = 192;
constexpr int WS_SMEM_BYTES = STAGES * STAGE_FL * 4 + 4 * 32 * 33 * 4 + 256;

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(mbar)) : "memory");
}

__global__ void __launch_bounds__(WS_THREADS, 1) kr_gemm(const GemmArgs g) {
  extern __shared__ __align__(1024) float krsm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int count = *g.count;
  const int nk = nkc(g.p), np = npairs(g.n4);
  const int mtiles = (count + BM - 1) / BM, ntiles = (np + BN - 1) / BN, tiles = mtiles * ntiles;
  if ((int)blockIdx.x >= tiles) return;
  float* stage = krsm;
  float* scr = krsm + STAGES * STAGE_FL;  // epilogue transpose scratch, [4 warps][32][33]
  uint64_t* full = reinterpret_cast<uint64_t*>(scr + 4 * 32 * 33);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tslot)),
                 "n"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(full + s, 1); tc::mbar_init(empty + s, 1); }
    for (int a = 0; a < 2; ++a) { tc::mbar_init(tfull + a, 1); tc::mbar_init(tempty + a, 4); }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 4) {
    if (lane == 0) {  // producer: four bulk copies per K chunk into the ring
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int mt = t % mtiles, nt = t / mtiles;
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) tc::mbar_wait(empty + s, ((it / STAGES) - 1) & 1);
          float* st = stage + s * STAGE_FL;
          mbar_expect_tx(full + s, STAGE_FL * 4);
          const long long ao = ((long long)mt * nk + kc) * A_FL, bo = ((long long)nt * nk + kc) * B_FL;
          bulk_g2s(st, g.whi + ao, A_FL * 4, full + s);
          bulk_g2s(st + A_FL, g.wlo + ao, A_FL * 4, full + s);
          bulk_g2s(st + 2 * A_FL, g.gghi + bo, B_FL * 4, full + s);
          bulk_g2s(st + 2 * A_FL + B_FL, g.gglo + bo, B_FL * 4, full + s);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issuer: 4 k-steps of 8 per chunk, three products each (3×TF32)
      const uint32_t idesc = idesc_256();
      int it = 0, li = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++li) {
        const int acc = li & 1;
        if (li >= 2) tc::mbar_wait(tempty + acc, ((li >> 1) - 1) & 1);  // the epilogue drained it
        tc::tc_fence_after();
        const uint32_t tacc = tmem + (uint32_t)(acc * BN);
        for (int kc = 0; kc < nk; ++kc, ++it) {
          const int s = it % STAGES;
          tc::mbar_wait(full + s, (it / STAGES) & 1);
          tc::tc_fence_after();
          const float* st = stage + s * STAGE_FL;
          const uint32_t ahi = tc::smem_u32(st), alo = tc::smem_u32(st + A_FL);
          const uint32_t bhi = tc::smem_u32(st + 2 * A_FL), blo = tc::smem_u32(st + 2 * A_FL + B_FL);
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            const uint32_t off = ks * 2 * 128;
            const uint32_t acc0 = (kc > 0 || ks > 0) ? 1u : 0u;
            tc::mma_tf32(tacc, tc::make_desc(ahi + off), tc::make_desc(bhi + off), idesc, acc0);
            tc::mma_tf32(tacc, tc::make_desc(ahi + off), tc::make_desc(blo + off), idesc, 1u);
            tc::mma_tf32(tacc, tc::make_desc(alo + off), tc::make_desc(bhi + off), idesc, 1u);
          }
          tc::commit(empty + s);
        }
        tc::commit(tfull + acc);
      }
    }
  } else {
    // ---- epilogue warps 0-3: warp w holds problems (slots) mt*128 + 32w + [0, 32) ----
    float* T = scr + warp * (32 * 33);
    const int n = g.n, n4 = g.n4, m = g.m;
    int li = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++li) {
      const int mt = t % mtiles, nt = t / mtiles, acc = li & 1;
      tc::mbar_wait(tfull + acc, (li >> 1) & 1);
      tc::tc_fence_after();
      __syncwarp();
      // lane r: problem of slot mt*128 + 32w + r (the batched engine's packed
      // layout is uniform, bnd_layout: a row's offset does not depend on the
      // problem's system size, so one offset per pair serves every problem)
      const int slot_l = mt * BM + 32 * warp + lane;
      const int nrow = min(32, count - (mt * BM + 32 * warp));  // warp-uniform (may be ≤ 0)
      int b_l = 0;
      float* stb_l = nullptr;
      if (lane < nrow) {
        b_l = g.slotmap[slot_l];
        stb_l = g.st + (long long)b_l * g.st_stride;
      }
      float dmx = 0.f;  // lane r: max |diag| of problem r over this tile's pairs
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(acc * BN + c0), v);
#pragma unroll
        for (int c = 0; c < 32; ++c) T[lane * 33 + c] = v[c];
        __syncwarp();
        if (nrow > 0) {
          const int tp = nt * BN + c0 + lane;  // lane = pair column
          const bool tok = tp < np;
          int i = 0, j = 0;
          if (tok) {
            i = (int)((sqrtf(8.f * tp + 1.f) - 1.f) * 0.5f);
            while ((i + 1) * (i + 2) / 2 <= tp) ++i;
            while (i * (i + 1) / 2 > tp) --i;
            j = tp - i * (i + 1) / 2;
          }
          const int bi = i >> 4, ti = i & 15;
          const int off = 128 * bi * (bi + 1) + 64 * bi + ti * (16 * bi + 20) + j;  // KLayout::make(.., true).off(i) + j
          const bool inner = tok && i < n && j < n, isdiag = tok && i == j && i < n;
          const bool anyd = __any_sync(0xffffffffu, isdiag);
          float q = 0.f;
          if (g.sQ == 0 && inner) q = __ldg(g.Q + (size_t)i * n + j);
          for (int r = 0; r < nrow; ++r) {
            const int b = __shfl_sync(0xffffffffu, b_l, r);
            float val = 0.f;
            if (tok) {
              const float qq = g.sQ == 0 ? q : (inner ? __ldg(g.Q + g.sQ * b + (size_t)i * n + j) : 0.f);
              val = inner ? qq + T[r * 33 + lane] : (i == j ? 1.f : 0.f);
              g.kw[(long long)b * g.kstride + off] = val;
            }
            if (anyd) {
              const float mx =
                  __uint_as_float(__reduce_max_sync(0xffffffffu, isdiag ? __float_as_uint(fabsf(val)) : 0u));
              if (lane == r) dmx = fmaxf(dmx, mx);
            }
          }
        }
        __syncwarp();
      }
      if (lane < nrow && dmx > 0.f) atomicMax(reinterpret_cast<int*>(stb_l) + 4, __float_as_int(dmx));  // BScal::dmax
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

}  // namespace kr
}  // namespace qpb

// tc_syrk.cuh — 5th-generation tensor cores (tcgen05) for the one part of the
// hot path that is a genuine dense contraction at large n: the KKT assembly
// H = Q + Gᵀ diag(ω) G, computed in an
// accuracy-preserving 3×TF32 split (a·b ≈ a_hi b_hi + a_hi b_lo + a_lo b_hi,
// hi = tf32(a), lo = tf32(a − hi)) so the result keeps f32 accuracy.
//
// One CTA computes 128×128 output tiles: operands are staged from global
// memory into shared memory in the canonical no-swizzle K-major UMMA layout
// (K-major: core matrix = 8 MN-rows × 16 B of K), one elected thread issues tcgen05.mma.kind::tf32 with the
// accumulator in TMEM (128 lanes × 128 fp32 columns), tcgen05.commit signals an
// mbarrier, and the four warps read their 32-lane quarter back with
// tcgen05.ld.32x32b for the epilogue.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qpb {
namespace tc {

constexpr int TM = 128;  // tile M (lanes)
constexpr int TN = 128;  // tile N (TMEM columns)
constexpr int TK = 32;   // K staged per round (4 MMA k-steps of 8)
// smem bytes per operand tile: 128 × 32 tf32 = 16 KB; four (A_hi, A_lo, B_hi, B_lo)
constexpr int OP_BYTES = TM * TK * 4;
constexpr int SMEM_BYTES = 4 * OP_BYTES + 64;  // + mbarrier and TMEM address

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// tf32(x) rounded to nearest, ties away from zero — cvt.rna.tf32.f32 for
// every finite x (and ±inf on overflow), as two integer operations: adding
// half a tf32 ulp to the magnitude bits and clearing the 13 low mantissa
// bits (ptxas expands cvt.rna.tf32 into a compare, add, mask and select;
// this halves the split work of the 3×TF32 staging loops)
__device__ __forceinline__ float to_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Canonical K-major, no swizzle: element (mn, k) of a TM×TK tile.  Core
// matrix = 8 MN-rows × 16 B (4 tf32 along K), 128 B contiguous; the TK/4 K
// chunks of one 8-row MN group are adjacent (LBO = 128 B), MN groups are
// TK/4 core matrices apart (SBO).  (MN-major operands read back as zeros for
// kind::tf32 on this part — measured by tools/tc_probe.py — so K-major it is.)
__device__ __forceinline__ int op_offset(int mn, int k) {
  return ((mn >> 3) * (TK / 4) + (k >> 2)) * 32 + (mn & 7) * 4 + (k & 3);  // in floats
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  const uint64_t lbo = 128 >> 4;
  const uint64_t sbo = (uint64_t)((TK / 4) * 128) >> 4;
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= lbo << 16;
  d |= sbo << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor: kind::tf32, D = f32, A = B = tf32, both K-major,
// N = TN, M = TM.
__device__ __forceinline__ uint32_t make_idesc() {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format = F32
  d |= 2u << 7;                    // a_format = TF32
  d |= 2u << 10;                   // b_format = TF32
  d |= (uint32_t)(TN >> 3) << 17;  // n_dim
  d |= (uint32_t)(TM >> 4) << 24;  // m_dim
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 consecutive fp32 TMEM columns of this thread's lane (warp w reads lanes 32w..32w+31)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared state of the tensor-core helper (lives at the start of `buf`).
struct TcState {
  float *ahi, *alo, *bhi, *blo;
  uint64_t* mbar;
  uint32_t* tmem_slot;   // TMEM base address (written by tcgen05.alloc)
  uint32_t* phase_slot;  // parity of the mbarrier phase the next commit completes
};

__device__ __forceinline__ TcState tc_state(void* buf) {
  TcState s;
  char* b = reinterpret_cast<char*>(buf);
  s.ahi = reinterpret_cast<float*>(b);
  s.alo = reinterpret_cast<float*>(b + OP_BYTES);
  s.bhi = reinterpret_cast<float*>(b + 2 * OP_BYTES);
  s.blo = reinterpret_cast<float*>(b + 3 * OP_BYTES);
  s.mbar = reinterpret_cast<uint64_t*>(b + 4 * OP_BYTES);
  s.tmem_slot = reinterpret_cast<uint32_t*>(b + 4 * OP_BYTES + 16);
  s.phase_slot = reinterpret_cast<uint32_t*>(b + 4 * OP_BYTES + 20);
  return s;
}

// TMEM: TN fp32 columns for one CTA.  Called by all threads (warp 0 allocates).
__device__ __forceinline__ uint32_t tmem_alloc(const TcState& s) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s.tmem_slot)),
                 "n"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(s.mbar, 1);
    *s.phase_slot = 0u;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *s.tmem_slot;
}

__device__ __forceinline__ void tmem_free(uint32_t taddr) {
  __syncthreads();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(TN));
}

// ------------------------------------------------------------------------
// Accumulate one 128×128 tile  C[i0+r][j0+c] = Σ_k G[k][i0+r] ω_k G[k][j0+c]
// (r, c < 128, rows/cols ≥ n treated as zero) and hand it to the epilogue
// `epi(row0, col, t)` in 32×32 blocks: lane l of a warp gets column col =
// c0 + l of rows row0 .. row0+31, value of row row0 + r at t[33 r] (so the
// lanes of a warp cover consecutive columns: coalesced global access).
// NT threads (multiple of 128).  The G values of K-chunk c+1 are loaded into
// registers while the tensor core works on chunk c.  TMEM address and
// mbarrier parity are kept in shared memory (tmem_alloc).  Ends with a
// barrier.
// ------------------------------------------------------------------------
template <int NT, typename Epi>
__device__ void syrk_tile(const TcState& s, const float* __restrict__ G, const float* om, int p, int n, int i0,
                          int j0, Epi epi) {
  static_assert(NT % 128 == 0, "syrk_tile: NT must be a multiple of 128");
  constexpr int U = (TK / 4) * TM / NT;  // 16-byte K-chunk rows staged per thread and operand
  const int tid = threadIdx.x;
  const uint32_t tmem = *s.tmem_slot;
  uint32_t phase = *s.phase_slot;  // read before the first barrier below; written after it
  const uint32_t idesc = make_idesc();
  float ra[U][4], rb[U][4];
  // one unit: one mn, 4 consecutive k (coalesced global reads across mn)
  auto load = [&](int k0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int unit = tid + u * NT, kc = unit / TM, mn = unit - kc * TM;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = k0 + 4 * kc + t;
        const bool kok = k < p;
        const float* g = G + (size_t)(kok ? k : 0) * n;
        ra[u][t] = (kok && i0 + mn < n) ? __ldg(g + i0 + mn) : 0.f;
        rb[u][t] = (kok && j0 + mn < n) ? __ldg(g + j0 + mn) : 0.f;  // ω applied in store()
      }
    }
  };
  auto store = [&](int k0) {  // ω, hi/lo split, conflict-free float4 stores in the K-major layout
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int unit = tid + u * NT, kc = unit / TM, mn = unit - kc * TM;
      float4 ah, al, bh, bl;
      float* pah = &ah.x; float* pal = &al.x; float* pbh = &bh.x; float* pbl = &bl.x;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = k0 + 4 * kc + t;
        const float bv = k < p ? om[k] * rb[u][t] : 0.f;
        pah[t] = to_tf32(ra[u][t]); pal[t] = to_tf32(ra[u][t] - pah[t]);
        pbh[t] = to_tf32(bv); pbl[t] = to_tf32(bv - pbh[t]);
      }
      const int o = op_offset(mn, 4 * kc);
      *reinterpret_cast<float4*>(s.ahi + o) = ah; *reinterpret_cast<float4*>(s.alo + o) = al;
      *reinterpret_cast<float4*>(s.bhi + o) = bh; *reinterpret_cast<float4*>(s.blo + o) = bl;
    }
  };
  load(0);
  for (int k0 = 0; k0 < p; k0 += TK) {
    store(k0);
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ahi = smem_u32(s.ahi), alo = smem_u32(s.alo), bhi = smem_u32(s.bhi), blo = smem_u32(s.blo);
      const uint32_t kstep = 2 * 128;  // bytes per MMA k-step of 8 (two K chunks)
#pragma unroll
      for (int ks = 0; ks < TK / 8; ++ks) {
        const uint32_t off = ks * kstep;
        const uint32_t acc0 = (k0 > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, make_desc(ahi + off), make_desc(bhi + off), idesc, acc0);
        mma_tf32(tmem, make_desc(ahi + off), make_desc(blo + off), idesc, 1u);
        mma_tf32(tmem, make_desc(alo + off), make_desc(bhi + off), idesc, 1u);
      }
      commit(s.mbar);
    }
    if (k0 + TK < p) load(k0 + TK);  // overlaps the MMAs of this chunk
    {
      // L2 prefetch of the G rows 3 chunks ahead (config 5's G, 8 MB per
      // problem, does not stay in L2): 32 rows × (4 + 4) 128-B lines of the
      // i0 and j0 column ranges, one line per thread and round
      const int kp = k0 + 3 * TK;
#pragma unroll
      for (int e = tid; e < TK * 8; e += NT) {
        const int r = e >> 3, sg = e & 7;
        const int k = kp + r, c = (sg < 4 ? i0 : j0) + 32 * (sg & 3);
        if (k < p && c < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(G + (size_t)k * n + c));
      }
    }
    mbar_wait(s.mbar, phase);
    phase ^= 1u;
    tc_fence_after();
  }
  if (tid == 0) *s.phase_slot = phase;
  // ---- epilogue: TMEM → registers → per-warp transpose in the (now free)
  //      operand buffers → coalesced row segments.  Warp w reads TMEM lane
  //      quarter w % 4; with NT = 256 the two warps of a quarter split the
  //      columns. ----
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int NH = NT / 128;
  const int q = warp & 3, half = warp >> 2;
  float* T = s.ahi + warp * (32 * 33);
#pragma unroll 1
  for (int c0 = half * (TN / NH); c0 < (half + 1) * (TN / NH); c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0, v);
#pragma unroll
    for (int c = 0; c < 32; ++c) T[lane * 33 + c] = v[c];
    __syncwarp();
    epi(i0 + 32 * q, j0 + c0 + lane, T + lane);
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
}

}  // namespace tc
}  // namespace qpb

namespace qpb {
namespace tc {

// Diagnostic kernel (qp_debug_tc_syrk): dense H = Q + Gᵀ diag(ω) G, n×n,
// through syrk_tile (all 128×128 tiles, upper ones too).  One CTA.
template <int NT>
__global__ void __launch_bounds__(NT, 1) debug_syrk_kernel(const float* G, const float* om, const float* Q, int n,
                                                          int p, float* H) {
  extern __shared__ __align__(128) unsigned char tcsm[];
  const TcState s = tc_state(tcsm);
  const uint32_t tmem = tmem_alloc(s);
  for (int i0 = 0; i0 < n; i0 += TM)
    for (int j0 = 0; j0 < n; j0 += TN)
      syrk_tile<NT>(s, G, om, p, n, i0, j0, [&](int row0, int col, const float* t) {
        for (int r = 0; r < 32; ++r) {
          const int row = row0 + r;
          if (row < n && col < n) H[(size_t)row * n + col] = Q[(size_t)row * n + col] + t[33 * r];
        }
      });
  tmem_free(tmem);
}

}  // namespace tc
}  // namespace qpb

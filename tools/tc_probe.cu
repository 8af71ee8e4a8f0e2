// Standalone probe of the tcgen05 building blocks in tc_syrk.cuh (diagnostic).
#include "../paper_2605_17913_b200/csrc/tc_syrk.cuh"
using namespace qpb::tc;

__device__ __forceinline__ void tmem_st1(uint32_t taddr, float x) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(x)) : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// mode 0: st/ld round trip. mode 1: MMA on A,B given (TM×8 each, [k][mn] dense) MN-major.
// out: 128×128 tile; info[0] = tmem addr, info[1] = spins
__global__ void probe(int mode, const float* A, const float* B, float* out, unsigned* info, uint64_t desc_xor,
                      uint32_t idesc_xor) {
  extern __shared__ __align__(128) unsigned char sm[];
  TcState s = tc_state(sm);
  uint32_t tmem = tmem_alloc(s);
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) info[0] = tmem;
  if (mode == 0) {
    for (int c = 0; c < 128; ++c) tmem_st1(tmem + ((32u * warp) << 16) + c, (float)(1000 * (32 * warp + lane) + c));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  } else {
    for (int e = tid; e < 8 * 128; e += 128) {
      int kk = e / 128, mn = e % 128;
      s.ahi[op_offset(mn, kk)] = A[e];
      s.bhi[op_offset(mn, kk)] = B[e];
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      mma_tf32(tmem, make_desc(smem_u32(s.ahi)) ^ desc_xor, make_desc(smem_u32(s.bhi)) ^ desc_xor,
               make_idesc() ^ idesc_xor, 0u);
      commit(s.mbar);
    }
    mbar_wait(s.mbar, 0);
    tc_fence_after();
  }
  for (int c0 = 0; c0 < 128; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((32u * warp) << 16) + c0, v);
    for (int c = 0; c < 32; ++c) out[(32 * warp + lane) * 128 + c0 + c] = v[c];
  }
  tmem_free(tmem);
}

extern "C" int run_probe(int mode, const float* A, const float* B, float* out, unsigned* info, unsigned long long dx,
                         unsigned ix) {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  probe<<<1, 128, SMEM_BYTES>>>(mode, A, B, out, info, dx, ix);
  return (int)cudaDeviceSynchronize();
}

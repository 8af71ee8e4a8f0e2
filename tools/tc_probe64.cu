// Probe: where does tcgen05.mma.cta_group::1.kind::tf32 with M = 64 put row m
// of D in TMEM?  A[m][0] = m + 1, B[n][0] = 1 (K-major, K = 8), N = 64.
#include "../paper_2605_17913_b200/csrc/tc_syrk.cuh"
using namespace qpb::tc;

__global__ void probe64(float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  TcState s = tc_state(sm);
  uint32_t tmem = tmem_alloc(s);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // clear TMEM columns 0..63 of every lane
  for (int c = 0; c < 64; ++c) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + ((32u * warp) << 16) + c),
                 "r"(__float_as_uint(-1.f)) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  // operands: 64 rows × TK(32) floats K-major (only k < 8 used)
  for (int e = tid; e < 64 * 8; e += 128) {
    const int m = e / 8, k = e % 8;
    s.ahi[op_offset(m, k)] = (k == 0) ? (float)(m + 1) : 0.f;
    s.bhi[op_offset(m, k)] = (k == 0) ? 1.f : 0.f;
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((64u >> 4) << 24);
    mma_tf32(tmem, make_desc(smem_u32(s.ahi)), make_desc(smem_u32(s.bhi)), idesc, 0u);
    commit(s.mbar);
  }
  mbar_wait(s.mbar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 64; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((32u * warp) << 16) + c0, v);
    for (int c = 0; c < 32; ++c) out[(32 * warp + lane) * 64 + c0 + c] = v[c];
  }
  tmem_free(tmem);
}

extern "C" int run_probe64(float* out) {
  cudaFuncSetAttribute(probe64, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  probe64<<<1, 128, SMEM_BYTES>>>(out);
  return (int)cudaDeviceSynchronize();
}

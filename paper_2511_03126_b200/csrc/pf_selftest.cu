// Diagnostic: one 128 x N x K bf16 GEMM through exactly the operand layouts, descriptors, MMA
// issue, commit and TMEM read-back the tile kernel uses (pf_tc.cuh). Lets the tests pin the
// tcgen05 plumbing against torch.matmul independently of the fusion logic.
#include <cuda_bf16.h>

#include "pf_common.cuh"
#include "pf_tc.cuh"

namespace pf {
namespace {

__global__ void __launch_bounds__(128, 1) k_umma_selftest(const uint16_t* __restrict__ A,
                                                          const uint16_t* __restrict__ B,
                                                          float* __restrict__ C, int K, int N,
                                                          int ts) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + 128 * K * 2;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;

  // A: thread m writes its row (K-major SW128)
  for (int k = 0; k < K; ++k)
    *reinterpret_cast<uint16_t*>(sA + tc::a_off(tid, k, 128)) = A[tid * K + k];
  // B: 16-byte chunks via cp.async (N-major SW128)
  const int qn = N / 8;
  for (int e = tid; e < K * qn; e += 128) {
    const int k = e / qn, q = e % qn;
    tc::cp_async16(tc::smem_u32(sB + tc::b_chunk_off(k, q, K)), B + (int64_t)k * N + q * 8);
  }
  tc::cp_async_wait_all();
  tc::fence_async_shared();
  if (tid == 0) tc::mbar_init(&mbar, 1);
  uint32_t ncols = 32;
  while (ncols < (uint32_t)N) ncols <<= 1;
  if (ts) ncols = 512;  // A lives at columns [256, 256 + K/2)
  if (warp == 0) tc::tmem_alloc(&tmem_base, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, N, false, true);
    // TS mode: A copied smem -> TMEM columns [256, 256 + K/2) once, then A read from TMEM
    const uint32_t ta = tbase + 256u;
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = tc::smem_desc_sw128(tc::smem_u32(sA) + (s >> 2) * 128 * 128 + (s & 3) * 32, 16, 1024);
      if (ts) tc::tmem_cp_128x256b(ta + (uint32_t)(s * 8), ad);
    }
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t ad = tc::smem_desc_sw128(tc::smem_u32(sA) + (s >> 2) * 128 * 128 + (s & 3) * 32, 16, 1024);
      const uint64_t bd = tc::smem_desc_sw128(tc::smem_u32(sB) + s * 2048, K * 128, 1024);
      if (ts)
        tc::mma_bf16_ts(tbase, ta + (uint32_t)(s * 8), bd, idesc, s > 0 ? 1u : 0u);
      else
        tc::mma_bf16(tbase, ad, bd, idesc, s > 0 ? 1u : 0u);
    }
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 32 && c0 + i < N; ++i) C[(int64_t)tid * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, ncols);
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_selftest_umma(const void* a, const void* b, float* c, int32_t k, int32_t n,
                                int32_t ts, void* stream) {
  if (k < 16 || k % 64 != 0 || k > 256 || n < 16 || n % 16 != 0 || n > 256 || (ts && n > 256 - 0))
    return set_error(PF_ERR_VALUE, "selftest_umma: need k in {64..256, %%64} and n in {16..256, %%16}");
  // B occupies whole 128-byte swizzle rows: ceil(n/64) halves of k rows x 128 B
  const size_t smem = 128 * (size_t)k * 2 + (size_t)((n + 63) / 64) * k * 128 + 1024;
  cudaFuncSetAttribute(k_umma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_umma_selftest<<<1, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint16_t*>(a), reinterpret_cast<const uint16_t*>(b), c, k, n, ts);
  return check_launch("selftest_umma");
}

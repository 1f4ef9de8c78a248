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

// ---- diagnostic: tcgen05.mma issue/execution rate (cycles per M=128 x N x K=16 MMA) -------------------
// One CTA per SM; thread 0 issues `reps` rounds of 8 MMAs (K = 128) on resident operands (B in
// shared memory, A in shared memory (ss) or TMEM (ts)) and times issue -> completion with clock64.
// `stores` != 0 makes warps 1-3 stream 16-byte shared-memory stores meanwhile (the tile kernel's
// cp.async traffic competes with the MMA's B reads for shared-memory bandwidth).
namespace pf {
namespace {
__global__ void __launch_bounds__(128, 1) k_umma_rate(int n, int ts, int reps, int stores,
                                                      unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int K = 128;
  unsigned char* sA = smem;                 // 128 x 128 bf16 (32 KB)
  unsigned char* sB = smem + 32768;         // K x n bf16, n/64 halves of K x 128 B
  unsigned char* sX = sB + (n / 64) * K * 128;  // store scratch (32 KB)
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (32768 + (n / 64) * K * 128) / 16; e += 128)
    reinterpret_cast<uint4*>(smem)[e] = make_uint4(0x3c003c00u, 0u, 0x3c003c00u, 0u);
  tc::fence_async_shared();
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    done = 0;
  }
  if (warp == 0) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (warp == 0 && ts == 2) {  // warp-uniform issue, elected lane
    const uint32_t idesc = tc::idesc_bf16_f32(128, n, false, true);
    const uint32_t ta = tbase + 256u;
    const uint32_t b0 = tc::smem_u32(sB);
    if (tid == 0) {
      for (int s = 0; s < K / 16; ++s)
        tc::tmem_cp_128x256b(ta + (uint32_t)(s * 8),
                             tc::smem_desc_sw128(tc::smem_u32(sA) + (s >> 2) * 128 * 128 + (s & 3) * 32, 16, 1024));
      tc::mma_commit(&mbar);
    }
    __syncwarp();
    tc::mbar_wait(&mbar, 0);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int s = 0; s < K / 16; ++s)
        tc::mma_bf16_ts_elect(tbase, ta + (uint32_t)(s * 8), tc::smem_desc_sw128(b0 + s * 2048, K * 128, 1024), idesc, 1u);
    }
    const long long t1 = clock64();
    tc::mma_commit_elect(&mbar);
    tc::mbar_wait(&mbar, 1);
    const long long t2 = clock64();
    if (tid == 0) {
      out[blockIdx.x * 2] = (unsigned long long)(t1 - t0);
      out[blockIdx.x * 2 + 1] = (unsigned long long)(t2 - t0);
      done = 1;
    }
  } else if (tid == 0 && ts != 2) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, n, false, true);
    const uint32_t ta = tbase + 256u;
    for (int s = 0; s < K / 16; ++s)
      tc::tmem_cp_128x256b(ta + (uint32_t)(s * 8),
                           tc::smem_desc_sw128(tc::smem_u32(sA) + (s >> 2) * 128 * 128 + (s & 3) * 32, 16, 1024));
    tc::mma_commit(&mbar);
    tc::mbar_wait(&mbar, 0);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < K / 16; ++s) {
        const uint64_t bd = tc::smem_desc_sw128(tc::smem_u32(sB) + s * 2048, K * 128, 1024);
        if (ts) {
          tc::mma_bf16_ts(tbase, ta + (uint32_t)(s * 8), bd, idesc, 1u);
        } else {
          const uint64_t ad = tc::smem_desc_sw128(tc::smem_u32(sA) + (s >> 2) * 128 * 128 + (s & 3) * 32, 16, 1024);
          tc::mma_bf16(tbase, ad, bd, idesc, 1u);
        }
      }
    const long long t1 = clock64();
    tc::mma_commit(&mbar);
    tc::mbar_wait(&mbar, 1);
    const long long t2 = clock64();
    out[blockIdx.x * 2] = (unsigned long long)(t1 - t0);
    out[blockIdx.x * 2 + 1] = (unsigned long long)(t2 - t0);
    done = 1;
  } else if (stores == 1 && warp > 0) {
    uint4* x = reinterpret_cast<uint4*>(sX);
    int i = tid;
    while (!done) {
      x[i & 2047] = make_uint4(i, i, i, i);
      i += 96;
    }
  } else if (stores == 2 && warp > 0) {
    // TMEM load latency under the MMA stream: tcgen05.ld 32x32b.x32 of columns 448.. + wait::ld
    const uint32_t ta = tbase + 448u + ((uint32_t)(32 * warp) << 16);
    long long cyc = 0;
    int cnt = 0;
    float acc = 0.f;
    while (!done) {
      float v[32];
      const long long a0 = clock64();
      tc::tmem_ld32(ta, v);
      cyc += clock64() - a0;
      ++cnt;
      acc += v[0];
    }
    if (tid == 32) {
      out[2 * gridDim.x + blockIdx.x * 2] = (unsigned long long)cyc;
      out[2 * gridDim.x + blockIdx.x * 2 + 1] = (unsigned long long)cnt + (acc == 12345.f ? 1 : 0);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, 512);
}
}  // namespace
}  // namespace pf

extern "C" int pf_bench_umma(int32_t n, int32_t ts, int32_t reps, int32_t stores, void* out_dev, void* stream) {
  if (n != 64 && n != 128 && n != 256) return set_error(PF_ERR_VALUE, "bench_umma: n in {64, 128, 256}");
  const size_t smem = 32768 + (size_t)(n / 64) * 128 * 128 + 32768 + 1024;
  cudaFuncSetAttribute(k_umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_umma_rate<<<sms, 128, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, ts, reps, stores, reinterpret_cast<unsigned long long*>(out_dev));
  return check_launch("bench_umma");
}

// ---- diagnostic: B-operand loader throughput, cp.async (tile kernel's loader pattern) vs TMA
// tile::gather4 (4 arbitrary 128-byte rows per op into the 128-byte-swizzled layout) ----------------------
#include <cuda.h>
#include <cudaTypedefs.h>
#ifndef PF_GATHER_ISSUERS
#define PF_GATHER_ISSUERS 4
#endif
#include <mutex>
namespace pf {
namespace {
__device__ __forceinline__ uint32_t bench_row(int b, int s, int r, int cells) {
  uint32_t h = (uint32_t)(b * 7919 + s * 131 + r) * 2654435761u;
  return (h >> 8) % (uint32_t)(cells < 20000 ? cells : 20000) + (uint32_t)(s / 64) * 97u % (uint32_t)cells;
}
__global__ void __launch_bounds__(192, 1) k_gather_rate(const __grid_constant__ CUtensorMap map, const uint16_t* src,
                                                        int cells, int stages_total, int mode,
                                                        unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kSt = 8, kRows = 128, kBytes = kRows * 128;
  __shared__ uint64_t bar[kSt];
  const int tid = threadIdx.x;
  if (tid == 0)
    for (int s = 0; s < kSt; ++s) tc::mbar_init(&bar[s], 1);
  __syncthreads();
  const long long t0 = clock64();
  if (mode == 0) {
    // cp.async: 192 threads, thread -> 16-byte column q of rows r0, r0 + 24, ...; 5 stages in flight
    const int q = tid & 7, r0 = tid >> 3;
    for (int s = 0; s < stages_total; ++s) {
      const uint32_t sb = tc::smem_u32(smem + (s % kSt) * kBytes);
      const uint32_t dst0 = sb + (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + (((q ^ (r0 & 7)) & 7) << 4));
#pragma unroll
      for (int j = 0; j < kRows / 24 + 1; ++j) {
        const int r = r0 + 24 * j;
        if (r < kRows) tc::cp_async16(dst0 + (uint32_t)j * 3072u, src + (int64_t)bench_row(blockIdx.x, s, r, cells) * 1024 + (s & 15) * 64 + q * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (s >= 4) asm volatile("cp.async.wait_group 4;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (mode == 2) {
    // TMA gather4 from 4 issuing threads (lane 0 of warps 0-3), row indices precomputed per stage
    // (no index arithmetic in the issue loop); each thread issues a quarter of a stage's gathers
    __shared__ int rows[kSt][kRows];
    const int w = tid >> 5;
    for (int s = 0; s < stages_total; ++s) {
      const int st = s % kSt;
      if (s >= kSt - 1) tc::mbar_wait(&bar[(s - (kSt - 1)) % kSt], (uint32_t)(((s - (kSt - 1)) / kSt) & 1));
      constexpr int kIss = 4 * PF_GATHER_ISSUERS / 4;
      if (w < kIss) {
        for (int r = (tid & 31); r < kRows / kIss; r += 32) rows[st][w * (kRows / kIss) + r] = (int)bench_row(blockIdx.x, s, w * (kRows / kIss) + r, cells);
        __syncwarp();
        if ((tid & 31) == 0) {
          const uint32_t sb = tc::smem_u32(smem + st * kBytes);
          if (w == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&bar[st])), "r"(kBytes) : "memory");
          const int c = (s & 15) * 64;
          const int* rr = rows[st] + w * (kRows / kIss);
          for (int g = 0; g < kRows / (4 * kIss); ++g)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                ::"r"(sb + (w * (kRows / (4 * kIss)) + g) * 512), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c),
                "r"(rr[4 * g]), "r"(rr[4 * g + 1]), "r"(rr[4 * g + 2]), "r"(rr[4 * g + 3]), "r"(tc::smem_u32(&bar[st]))
                : "memory");
        }
      }
    }
    if (tid == 0)
      for (int s = stages_total - (kSt - 1); s < stages_total; ++s)
        if (s >= 0) tc::mbar_wait(&bar[s % kSt], (uint32_t)((s / kSt) & 1));
  } else if (tid == 0) {
    // TMA gather4: one thread; 7 stages in flight
    for (int s = 0; s < stages_total; ++s) {
      const int st = s % kSt;
      if (s >= kSt - 1) tc::mbar_wait(&bar[(s - (kSt - 1)) % kSt], (uint32_t)(((s - (kSt - 1)) / kSt) & 1));
      const uint32_t sb = tc::smem_u32(smem + st * kBytes);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(&bar[st])), "r"(kBytes) : "memory");
      for (int g = 0; g < kRows / 4; ++g) {
        const int c = (s & 15) * 64;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(sb + g * 512), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c),
            "r"((int)bench_row(blockIdx.x, s, 4 * g, cells)), "r"((int)bench_row(blockIdx.x, s, 4 * g + 1, cells)),
            "r"((int)bench_row(blockIdx.x, s, 4 * g + 2, cells)), "r"((int)bench_row(blockIdx.x, s, 4 * g + 3, cells)),
            "r"(tc::smem_u32(&bar[st]))
            : "memory");
      }
    }
    for (int s = stages_total - (kSt - 1); s < stages_total; ++s)
      if (s >= 0) tc::mbar_wait(&bar[s % kSt], (uint32_t)((s / kSt) & 1));
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace
}  // namespace pf

extern "C" int pf_bench_gather(const void* src_bf16, int32_t cells, int32_t stages, int32_t mode, void* out_dev,
                               void* stream) {
  using namespace pf;
  CUtensorMap m;
  auto fn = encode_tiled();
  if (!fn) return set_error(PF_ERR_CUDA, "bench_gather: no cuTensorMapEncodeTiled");
  const cuuint64_t dims[2] = {1024u, (cuuint64_t)cells};
  const cuuint64_t strides[1] = {2048u};
  const cuuint32_t box[2] = {64u, 1u};
  const cuuint32_t estr[2] = {1u, 1u};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src_bf16), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return set_error(PF_ERR_CUDA, "bench_gather: tensor map encode failed");
  const size_t smem = 8 * 128 * 128 + 1024;
  cudaFuncSetAttribute(k_gather_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_gather_rate<<<sms, 192, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      m, reinterpret_cast<const uint16_t*>(src_bf16), cells, stages, mode, reinterpret_cast<unsigned long long*>(out_dev));
  return check_launch("bench_gather");
}

// G = fmap @ text^T on the tensor cores for the bf16 tile path (the per-object table behind the
// similarity-by-associativity, see pf_tile.cu): one CTA per 128 feature cells, K = D streamed in
// 64-channel chunks through a 3-stage cp.async ring, tcgen05.mma (M=128, N=kpadg, K=16) into TMEM,
// epilogue writes G in bf16 (cells x kpadg, the tile kernel's S operand) and fp32 (cells x kpad,
// the SIMT overflow path). The text rows are rounded to bf16 once (k_text_bf16; bf16-feature mode
// bar 1e-2) and streamed with cp.async like the map rows; the MMAs are issued warp-uniformly.
#include <cuda_bf16.h>

#include "pf_common.cuh"
#include "pf_tc.cuh"
#include "pf_tile.cuh"

namespace pf {
namespace tile {
namespace {

constexpr int kGM = 128;     // cells per CTA
constexpr int kGStages = 3;  // cp.async ring depth (2 CTAs per SM)

__device__ __forceinline__ int lane_of(int tid) { return tid & 31; }

__global__ void k_text_bf16(const float* __restrict__ text, int k, int kpadg, int d, uint16_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)kpadg * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / d;
    out[e] = __bfloat16_as_ushort(__float2bfloat16_rn(n < k ? text[e] : 0.f));
  }
}

// softmax exponent bound of the tile epilogue: out[0] = max_k |t_k| (fp32, the rows exactly as the
// caller passed them: QueryTables does not normalise, grounding.py:86-93 does it upstream). NaN rows
// give NaN (the epilogue then takes the per-row max path and flags the NaN similarities).
__global__ void k_text_bound(const float* __restrict__ text, int k, int d, float* __restrict__ out) {
  __shared__ float wmax[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float m = 0.f;
  for (int r = warp; r < k; r += blockDim.x >> 5) {
    float ss = 0.f;
    for (int c = lane; c < d; c += 32) ss = fmaf(text[(int64_t)r * d + c], text[(int64_t)r * d + c], ss);
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float nr = sqrtf(ss);
    m = (nr > m || nr != nr) ? nr : m;  // NaN sticks
  }
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = (wmax[w] > r || wmax[w] != wmax[w]) ? wmax[w] : r;
    out[0] = r;
  }
}

// text rows -> bf16 hi and lo (x - hi) parts, rows >= k zero (x3 mode)
__global__ void k_text_split(const float* __restrict__ text, int k, int kpadg, int d, uint16_t* __restrict__ hi,
                             uint16_t* __restrict__ lo) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)kpadg * d;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / d;
    const float x = n < k ? text[e] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[e] = __bfloat16_as_ushort(h);
    lo[e] = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(h)));
  }
}

// X3 (f32 maps): stages hold the hi and lo parts of both operands and each K=16 step issues
// hi.hi + hi.lo + lo.hi; the epilogue also writes the lo part of G (Gbf_lo)
template <bool X3>
__global__ void __launch_bounds__(128) k_gproj_tc(const uint16_t* __restrict__ fmap, int64_t cells, int d,
                                                     const uint16_t* __restrict__ textbf, int k, int kpadg,
                                                     int kpad, uint16_t* __restrict__ Gbf,
                                                     float* __restrict__ G32, const uint16_t* __restrict__ fmap_lo,
                                                     const uint16_t* __restrict__ text_lo,
                                                     uint16_t* __restrict__ Gbf_lo) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // stage s: A [128 rows x 64 ch] (16 KB, K-major SW128) then B [kpadg rows x 64 ch] (K-major SW128)
  const int b_bytes = kpadg * 128;
  const int part_bytes = 16384 + b_bytes;  // [A | B] of one precision part
  const int stage_bytes = X3 ? 2 * part_bytes : part_bytes;
  __shared__ uint64_t mbar[kGStages];  // MMA completion per ring stage
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * kGM;
  const int nchunk = d / 64;
  const int nk = (k + 15) & ~15;  // MMA N: the materials rounded up to 16 (columns >= nk of G are 0)

  auto load = [&](int ch, int st) {
#pragma unroll
    for (int part = 0; part < (X3 ? 2 : 1); ++part) {
      unsigned char* sa = smem + st * stage_bytes + part * part_bytes;
      unsigned char* sb = sa + 16384;
      const uint16_t* fa = part ? fmap_lo : fmap;
      const uint16_t* fb = part ? text_lo : textbf;
      // A: row r, 16-byte piece q (8 channels): K-major SW128, one 64-channel atom column
      for (int e = tid; e < kGM * 8; e += 128) {
        const int r = e >> 3, q = e & 7;
        const int64_t cell = c0 + r < cells ? c0 + r : cells - 1;
        const uint32_t off = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((q ^ (r & 7)) & 7) << 4));
        tc::cp_async16(tc::smem_u32(sa + off), fa + cell * d + ch * 64 + q * 8);
      }
      // B: material n, channels ch*64 .. +64 (bf16 text, K-major SW128)
      for (int e = tid; e < nk * 8; e += 128) {
        const int n = e >> 3, q = e & 7;
        const uint32_t off = (uint32_t)((n >> 3) * 1024 + (n & 7) * 128 + (((q ^ (n & 7)) & 7) << 4));
        tc::cp_async16(tc::smem_u32(sb + off), fb + (int64_t)n * d + ch * 64 + q * 8);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  if (tid < kGStages) tc::mbar_init(&mbar[tid], 1);
  uint32_t ncols = 32;
  while (ncols < (uint32_t)nk) ncols <<= 1;
  if (warp == 0) tc::tmem_alloc(&tmem_base_s, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base_s;
  const uint32_t idesc = tc::idesc_bf16_f32(128, nk, false, false);

  // 3-stage ring: chunks ch+1 and ch+2 are in flight while chunk ch's MMAs run
  for (int c = 0; c < kGStages - 1 && c < nchunk; ++c) load(c, c);
  for (int ch = 0; ch < nchunk; ++ch) {
    const int st = ch % kGStages;
    if (ch + 1 < nchunk) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    tc::fence_async_shared();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) {  // warp-uniform issue, elected lane (scripts/umma_rate.py)
      const uint32_t a0 = tc::smem_u32(smem + st * stage_bytes), b0 = a0 + 16384;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t ad = tc::smem_desc_sw128(a0 + s * 32, 16, 1024);
        const uint64_t bd = tc::smem_desc_sw128(b0 + s * 32, 16, 1024);
        tc::mma_bf16_ss_elect(tbase, ad, bd, idesc, (ch | s) ? 1u : 0u);
        if constexpr (X3) {
          const uint64_t adl = tc::smem_desc_sw128(a0 + part_bytes + s * 32, 16, 1024);
          const uint64_t bdl = tc::smem_desc_sw128(b0 + part_bytes + s * 32, 16, 1024);
          tc::mma_bf16_ss_elect(tbase, ad, bdl, idesc, 1u);
          tc::mma_bf16_ss_elect(tbase, adl, bd, idesc, 1u);
        }
      }
      tc::mma_commit_elect(&mbar[st]);
    }
    // chunk ch+2 refills the stage of chunk ch-1 once that chunk's MMAs have completed
    if (ch + kGStages - 1 < nchunk) {
      if (ch >= 1) tc::mbar_wait(&mbar[(ch - 1) % kGStages], (uint32_t)(((ch - 1) / kGStages) & 1));
      load(ch + kGStages - 1, (ch + kGStages - 1) % kGStages);
    }
  }
  tc::mbar_wait(&mbar[(nchunk - 1) % kGStages], (uint32_t)(((nchunk - 1) / kGStages) & 1));
  tc::fence_after_sync();
  // epilogue through shared memory (the ring is free): TMEM row -> smem row, then each warp writes
  // whole rows of G (coalesced) instead of every thread striding through its own row
  float* srow = reinterpret_cast<float*>(smem);  // [128][kpadg + 1]
  const int ld = kpadg + 1;
  for (int cc = 0; cc < kpadg; cc += 32) {
    float v[32];
    if (cc < nk) {
      tc::tmem_ld32(tbase + ((uint32_t)(warp * 32) << 16) + cc, v);
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = 0.f;
    }
#pragma unroll
    for (int q = 0; q < 32; ++q) srow[tid * ld + cc + q] = cc + q < nk ? v[q] : 0.f;
  }
  __syncthreads();
  for (int r = warp; r < kGM; r += 4) {
    const int64_t cell = c0 + r;
    if (cell >= cells) break;
    for (int c = lane_of(tid); c < kpadg; c += 32) {
      const float val = srow[r * ld + c];
      const __nv_bfloat16 h = __float2bfloat16_rn(val);
      Gbf[cell * kpadg + c] = __bfloat16_as_ushort(h);
      if constexpr (X3) Gbf_lo[cell * kpadg + c] = __bfloat16_as_ushort(__float2bfloat16_rn(val - __bfloat162float(h)));
      if (G32 && c < kpad) G32[cell * kpad + c] = c < k ? val : 0.f;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tbase, ncols);
}

}  // namespace

int run_text_bound(const float* text, int k, int d, float* out, cudaStream_t st) {
  k_text_bound<<<1, 1024, 0, st>>>(text, k, d, out);
  return check_launch("text_bound");
}

int run_gproj_tc(const void* fmap, int64_t cells, int d, const float* text, int k, int kpadg, int kpad,
                 uint16_t* Gbf, float* G32, uint16_t* textbf, cudaStream_t st) {
  if (d % 64 != 0 || kpadg % 16 != 0 || kpadg > 256) return -1;
  k_text_bf16<<<grid_for((int64_t)kpadg * d, 256), 256, 0, st>>>(text, k, kpadg, d, textbf);
  if (int rc = check_launch("text_bf16")) return rc;
  const size_t smem = kGStages * (16384 + (size_t)kpadg * 128) + 1024;
  cudaFuncSetAttribute(k_gproj_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)((cells + kGM - 1) / kGM);
  k_gproj_tc<false><<<grid, 128, smem, st>>>(reinterpret_cast<const uint16_t*>(fmap), cells, d, textbf, k, kpadg,
                                             kpad, Gbf, G32, nullptr, nullptr, nullptr);
  return check_launch("gproj_tc");
}

int run_gproj_tc_x3(const uint16_t* fhi, const uint16_t* flo, int64_t cells, int d, const float* text, int k,
                    int kpadg, int kpad, uint16_t* Gbf, uint16_t* Gbf_lo, float* G32, uint16_t* text_hi,
                    uint16_t* text_lo, cudaStream_t st) {
  if (d % 64 != 0 || kpadg % 16 != 0 || kpadg > 256) return set_error(PF_ERR_VALUE, "gproj_x3: bad shapes");
  k_text_split<<<grid_for((int64_t)kpadg * d, 256), 256, 0, st>>>(text, k, kpadg, d, text_hi, text_lo);
  if (int rc = check_launch("text_split")) return rc;
  const size_t smem = kGStages * 2 * (16384 + (size_t)kpadg * 128) + 1024;
  cudaFuncSetAttribute(k_gproj_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const unsigned grid = (unsigned)((cells + kGM - 1) / kGM);
  k_gproj_tc<true><<<grid, 128, smem, st>>>(fhi, cells, d, text_hi, k, kpadg, kpad, Gbf, G32, flo, text_lo, Gbf_lo);
  return check_launch("gproj_tc_x3");
}

}  // namespace tile
}  // namespace pf

// Gram formulation of the bf16 fused query (the production tile kernel for bf16 maps).
//
// The similarity needs only two per-point quantities from the D-wide fused feature
// F_r = sum_t W[r,t] f_t (t over the tile's bilinear taps, fusion.py:65-93):
//   the numerators  S[r,k] = sum_t W[r,t] G[t,k]          (G = fmap . text^T, per cell: pf_gproj.cu)
//   the squared norm |F_r|^2 = sum_{t,t'} W[r,t] W[r,t'] <f_t, f_t'> = w_r^T M w_r
// with M = T T^T the Gram matrix of the tile's tap rows T (kt x D). A tile of 512 points spans a
// small fraction of a feature cell in every view, so its tap union is barely larger than a 128-point
// tile's (C5: ~128 vs ~112 taps, scripts/tile_taps_study.py). The D-wide work per tile is then one
// kt x kt x D Gram product instead of a 512 x kt x D feature product: per point the tensor work
// drops from 2 kt (D + K) to 2 kt^2 D / 512 + 2 kt (kt + K) and the L2 -> SMEM tap traffic from
// kt (D + K) / 128 to kt (D + K) / 512 rows of 2 bytes.
//
// Per work item (a 512-row tile, or a 128 / 32-row split of an overflowing one; <= 192 taps):
//   1. loaders gather the kt tap rows in 64-channel chunks into a 4-stage ring (cp.async, SW128),
//      then the tap rows of the bf16 G table (2 chunks of 64 materials);
//   2. MMA warp: Gram = T T^T on tcgen05 (A = B = the same K-major chunk; taps 128.. as a second
//      M block restricted to the lower-right corner), into TMEM;
//   3. accumulator warps drain the Gram to shared memory as bf16 M~ (rows 128.. rebuilt from the
//      transpose of block 0), the B operand of step 4;
//   4. per 128-row block b: builders write W_b (bilinear weights, bf16) straight into TMEM; the MMA
//      warp issues S_b = W_b G_taps and Y_b = W_b M~ (A from TMEM);
//   5. accumulator warps: |F_r|^2 = sum_t W[r,t] Y[r,t], then the same fused epilogue as k_tile_ws
//      (cosine, temperature softmax, regression, voxel atomics, integrate partials).
// The bf16 rounding of M~ changes |F| by ~1e-4 relative at C5 (scripts/gram_precision.py), well
// inside the bf16-feature bar of 1e-2.
//
// Warp roles (24 warps, setmaxnreg 48 / 144): 0-2 and 4-7 loaders, 3 MMA, 8-15 builders (two per
// TMEM lane quarter, view parity), 16-23 accumulators (two per lane quarter, material halves).
// TMEM (512 columns): region R [0, 320) holds the Gram (block 0 at 0, block 1 at 192) or one row
// block's S (0..127) and Y (128..319); W buffers at 320 and 416 (96 columns of bf16 pairs each).
// Work items come from a device-built list sorted by cost (k_collect_work, k_sort_work); CTA c takes
// list positions c, 2G - 1 - c, 2G + c, ... The C5 timing history and the variants measured and
// dropped are in profiles/r02_notes.md.
#include <type_traits>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "pf_common.cuh"
#include "pf_tc.cuh"
#include "pf_tile.cuh"
#include "pf_tile_dev.cuh"

namespace pf {
namespace tile {
namespace {

#ifndef PF_GRAM_BUILD_GROUPS
#define PF_GRAM_BUILD_GROUPS 2  // 8 builder warps (3 groups with 3 loader warps was measured slower)
#endif
#ifndef PF_GRAM_LOAD_WARPS
#define PF_GRAM_LOAD_WARPS 7
#endif
#ifndef PF_GRAM_REG_ACC
#define PF_GRAM_REG_ACC 144
#endif
// warps 0-2 and 4 .. kBuildWarp0-1: tap-row loaders; warp 3: MMA issuer; kBuildWarp0 ..: W builders
// (kBuildGroups per TMEM lane quarter); the last 8 warps: accumulators (two per lane quarter)
constexpr int kBuildGroups = PF_GRAM_BUILD_GROUPS;
constexpr int kBuildWarps = 4 * kBuildGroups;
constexpr int kLoadWarps = PF_GRAM_LOAD_WARPS;
constexpr int kBuildWarp0 = kLoadWarps + 1;
constexpr int kLoadThreads = 32 * kLoadWarps;
constexpr int kMmaWarp = 3;
constexpr int kBuildThreads = 32 * kBuildWarps;
constexpr int kAccWarp0 = kBuildWarp0 + kBuildWarps;
constexpr int kAccThreads = 256;
constexpr int kThreads = 32 * (kAccWarp0 + 8);
constexpr float kAffineR = 12e-3f;  // blocks wider than 2 kAffineR build with the exact projection
constexpr int kKt = kGramKt;        // taps per work item
constexpr int kStageBytes = kKt * 128;
constexpr int kStages = 4;          // ring depth (even: the two G chunks of an item are adjacent)
constexpr int kChunkBytes = kKt * 128;   // one 64-tap K chunk of M~ (kKt rows x 128 B)
constexpr int kMtBytes = 3 * kChunkBytes;
constexpr int kRowStep = kLoadThreads / 8;
constexpr int kRowsPer = (kKt + kRowStep - 1) / kRowStep;
constexpr int kHalfK = kMaxKpadTC / 2;
constexpr int kRegProducer = 48, kRegAcc = PF_GRAM_REG_ACC;
// registers per thread at launch (the pool setmaxnreg redistributes): 64K / threads, multiple of 8
constexpr int kRegLaunch = (65536 / kThreads) & ~7;
constexpr uint32_t kColS = 0, kColY = 128, kColG0 = 0, kColG1 = 192, kColW = 320, kWCols = kKt / 2;
static_assert(kColY + kKt <= kColW && kColW + 2 * kWCols <= 512, "TMEM budget");
static_assert(kRowsPer * kRowStep >= kKt, "loader rows");
static_assert((kThreads - kAccThreads) * (kRegLaunch - kRegProducer) >= kAccThreads * (kRegAcc - kRegLaunch),
              "register pool");
static_assert(kBuildWarp0 % 4 == 0 && kAccWarp0 % 4 == 0, "TMEM lane quarter = warp % 4");
static_assert(kStages % 2 == 0, "G chunk pairs never wrap the ring");

// PF_GRAM_TRAP (nvcc -DPF_GRAM_TRAP): every mbarrier wait traps after ~2 s instead of hanging
#ifdef PF_GRAM_TRAP
#define GWAIT(bar, par) tc::mbar_wait_or_trap(bar, par, __LINE__)
#define GWAIT_SLEEP(bar, par, ns) tc::mbar_wait_or_trap(bar, par, __LINE__)
#else
#define GWAIT(bar, par) tc::mbar_wait(bar, par)
#define GWAIT_SLEEP(bar, par, ns) tc::mbar_wait_sleep<ns>(bar, par)
#endif
#ifndef PF_GRAM_SLEEP_NS
#define PF_GRAM_SLEEP_NS 100
#endif
// PROF instantiation (PF_WS_DEBUG=1): cycles spent in each wait site, per CTA (printed by the host):
// 0 load:b_empty 1 mma:r_empty(gram) 2 mma:b_full(gram) 3 mma:b_full(G) 4 mma:a_full 5 mma:r_empty(blk)
// 6 build:a_empty 7 acc:r_full(gram) 8 acc:r_full(blk); 9 build busy, 10 acc busy, 11 total
// all other waits back off with a short sleep (PF_GRAM_WAIT_NS; 0 = spin): a spinning warp takes issue
// slots from the builders and accumulators on its SM sub-partition
#ifndef PF_GRAM_WAIT_NS
#define PF_GRAM_WAIT_NS 32
#endif
#if PF_GRAM_WAIT_NS > 0 && !defined(PF_GRAM_TRAP)
#undef GWAIT
#define GWAIT(bar, par) tc::mbar_wait_sleep<PF_GRAM_WAIT_NS>(bar, par)
#endif
#define GWAITP(bar, par, slot)                 \
  do {                                          \
    if constexpr (PROF) {                       \
      const long long t0_ = clock64();          \
      GWAIT(bar, par);                          \
      const long long t1_ = clock64();          \
      wcyc[slot] += t1_ - t0_;                  \
      tmark += t1_ - t0_;                       \
    } else {                                    \
      GWAIT(bar, par);                          \
    }                                           \
  } while (0)

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}

struct GramShared {
  uint64_t a_full[2], a_empty[2];
  uint64_t b_full[kStages], b_empty[kStages];
  uint64_t r_full, r_empty;
  uint32_t tmem_base;
  int pad;
  int32_t cell[2][kKt];
  ViewF sv[kMaxViewsTC];
  float4 vpk[kMaxViewsTC][5];
  int4 wlist[kBuildWarps][kMaxViewsTC / kBuildGroups + 1];      // builders: per-warp view list (per item)
  float4 wcoef[kBuildWarps][2 * (kMaxViewsTC / kBuildGroups + 1)];  // builders: per-warp expansion coefficients
  float4 yp[kMaxKpadTC];
  float4 yq[3][kMaxKpadTC / 4];  // per 4 materials: property 0, property 1, mid_theta (the 4-wide softmax loop)
  float2 yv2[kMaxKpadTC];
  float xss[2][2][kTile];  // [block parity][half][row]: double-buffered, so a block needs no closing barrier
  float xm[2][2][kTile];
  float xsum[2][2][6][kTile];
  double red[kMaxKpadTC + 8];
};

__device__ __forceinline__ uint4 ld_pref_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_pref_u2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_pref_f4(const void* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float warp_reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const float keep = up ? v[j + o] : v[j];
      const float send = up ? v[j] : v[j + o];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}
// the two accumulator warps of TMEM lane quarter qd (the same 32 rows, the two material halves)
// exchange per-row values through shared memory: a 64-thread named barrier per quarter (ids 4-7)
__device__ __forceinline__ void acc_pair_sync(int qd) {
  asm volatile("bar.sync %0, 64;" ::"r"(4 + qd) : "memory");
}
// reduce-scatter of 32 bf16 pairs over the warp (packed bf16x2 adds): lane l returns pair l summed
// over the 32 lanes
__device__ __forceinline__ uint32_t warp_reduce_scatter32_bf16x2(uint32_t (&a)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const uint32_t keep = up ? a[j + o] : a[j], send = up ? a[j] : a[j + o];
      const uint32_t x = __shfl_xor_sync(0xffffffffu, send, o);
      __nv_bfloat162 k2 = *reinterpret_cast<const __nv_bfloat162*>(&keep);
      const __nv_bfloat162 x2 = *reinterpret_cast<const __nv_bfloat162*>(&x);
      k2 = __hadd2(k2, x2);
      a[j] = *reinterpret_cast<const uint32_t*>(&k2);
    }
  }
  return a[0];
}
// two independent reduce-scatters interleaved level by level (twice the shuffles in flight)
__device__ __forceinline__ void warp_reduce_scatter32x2(float (&a)[32], float (&b)[32], int lane, float& ra, float& rb) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const float ka = up ? a[j + o] : a[j], sa = up ? a[j] : a[j + o];
      const float kb = up ? b[j + o] : b[j], sb = up ? b[j] : b[j + o];
      const float xa = __shfl_xor_sync(0xffffffffu, sa, o), xb = __shfl_xor_sync(0xffffffffu, sb, o);
      a[j] = ka + xa;
      b[j] = kb + xb;
    }
  }
  ra = a[0];
  rb = b[0];
}
// 16 columns of this warp's lanes (bf16 pairs of W)
// a 32-column Y chunk and the matching 16 columns of W (bf16 pairs) under one wait
__device__ __forceinline__ void tmem_ld_yw(uint32_t ty, uint32_t tw, uint32_t (&y)[32], uint32_t (&w)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%48];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47}, [%49];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(y[0]), "=r"(y[1]), "=r"(y[2]), "=r"(y[3]), "=r"(y[4]), "=r"(y[5]), "=r"(y[6]), "=r"(y[7]), "=r"(y[8]), "=r"(y[9]), "=r"(y[10]), "=r"(y[11]), "=r"(y[12]), "=r"(y[13]), "=r"(y[14]), "=r"(y[15]), "=r"(y[16]), "=r"(y[17]), "=r"(y[18]), "=r"(y[19]), "=r"(y[20]), "=r"(y[21]), "=r"(y[22]), "=r"(y[23]), "=r"(y[24]), "=r"(y[25]), "=r"(y[26]), "=r"(y[27]), "=r"(y[28]), "=r"(y[29]), "=r"(y[30]), "=r"(y[31]), "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(ty), "r"(tw)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16u(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&b2);
}
// byte offset of 16-byte piece q (taps 8q..8q+7 of K chunk j) of M~ row n (K-major SW128)
__device__ __forceinline__ uint32_t mt_off(int n, int j, int q) {
  return (uint32_t)(j * kChunkBytes + (n >> 3) * 1024 + (n & 7) * 128 + (((q ^ n) & 7) << 4));
}

__device__ __forceinline__ int ktp_ok(int kt, bool& ok) {
  const int ktp = (kt + 15) & ~15;
  ok = kt > 0 && ktp <= kKt;
  return ktp;
}
__device__ __forceinline__ int4 ld_pref_i4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// the k-th item of this CTA: the list is sorted by tap count, descending (k_sort_work), and CTA c
// takes positions c, 2G - 1 - c, 2G + c, ... (boustrophedon), so every CTA gets a similar mix of
// heavy and light items (a plain stride left the slowest CTA 3 % behind the mean at C5)
__device__ __forceinline__ int4 item_at(const TileParams& P, int nwork, int k) {
  const int g = gridDim.x, c = blockIdx.x;
  const int i = k * g + ((k & 1) ? g - 1 - c : c);
  return i < nwork ? ld_pref_i4(P.work + i) : make_int4(-1, 0, 0, 0);
}
// work-list entry {item, first row, rows | taps << 16, -}
__device__ __forceinline__ int e_rows(const int4& e) { return e.z & 0xffff; }
__device__ __forceinline__ int e_kt(const int4& e) { return e.z >> 16; }
__device__ __forceinline__ int e_nb(const int4& e) { return (e_rows(e) + 127) >> 7; }
// window shape class of a descriptor: 0: 2x2, 1: 3x2, 2: 2x3, 3: 3x3, 4: other, -1: no taps
__device__ __forceinline__ int shape_cls(uint2 d) {
  const int w = d.y & 0xff, h = (d.y >> 8) & 0xff;
  if (!w) return -1;
  return (w == 2 && h == 2) ? 0 : (w == 3 && h == 2) ? 1 : (w == 2 && h == 3) ? 2 : (w == 3 && h == 3) ? 3 : 4;
}

template <bool OUTS, bool PROF>
__global__ void __launch_bounds__(kThreads, 1) k_tile_gram(const __grid_constant__ TileParams P) {
  long long wcyc[24];
#pragma unroll
  for (int q = 0; q < 24; ++q) wcyc[q] = 0;
  const long long t_start = PROF ? clock64() : 0;
  long long tmark = t_start;
  // PROF phase timer: cycles since the previous mark into slot q
#define PT(q)                                   \
  do {                                          \
    if constexpr (PROF) {                       \
      const long long t_ = clock64();           \
      wcyc[q] += t_ - tmark;                    \
      tmark = t_;                               \
    }                                           \
  } while (0)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sB = smem;                          // kStages x [kKt rows x 128 B]
  unsigned char* sM = smem + kStages * kStageBytes;  // M~: 3 K chunks x [kKt rows x 128 B]
  __shared__ GramShared S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nd = P.d >> 6;
  const int nwork = *P.work_count;
  unsigned long long t_cta0 = 0;  // PF_GRAM_CTATIME: per-CTA start / end (%globaltimer, ns)
  if (P.ctatime && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_cta0));

  // ---- setup (as k_tile_ws) ----------------------------------------------------------------------
  for (int j = tid; j < P.nv; j += kThreads) {
    const ViewF w = make_viewf(P.views[j], P.d);
    S.sv[j] = w;
    S.vpk[j][0] = make_float4(w.R[0], w.R[1], w.R[2], w.t[0]);
    S.vpk[j][1] = make_float4(w.R[3], w.R[4], w.R[5], w.t[1]);
    S.vpk[j][2] = make_float4(w.R[6], w.R[7], w.R[8], w.t[2]);
    S.vpk[j][3] = make_float4(w.fx, w.cx, w.fy, w.cy);
    S.vpk[j][4] = make_float4(w.ru, w.rv, (float)(w.Wf - 1), (float)(w.Hf - 1));
  }
  for (int j = tid; j < kMaxKpadTC; j += kThreads) {
    float y[4];
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) y[pp] = (pp < P.p && j < P.k) ? P.values[j * P.p + pp] : 0.f;
    S.yv2[j] = make_float2(y[2], y[3]);
  }
  // softmax shift: see k_tile_ws (constant bound c = max_k |t_k| / T, or the row max when 2c > 120)
  const float cbound = 1.05f * __ldg(P.tbound) * P.inv_temp * 1.4426950408889634f;
  const int need_max = (2.f * cbound <= 120.f) ? 0 : 1;
  const float shift = need_max ? 0.f : -cbound;
  for (int j = tid; j < kMaxKpadTC / 2; j += kThreads) {
    auto val = [&](int kk, int pp) { return (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f; };
    const int a = 2 * j, b = 2 * j + 1;
    S.yp[2 * j] = make_float4(val(a, 0), val(b, 0), val(a, 1), val(b, 1));
    S.yp[2 * j + 1] = make_float4(a < P.k ? P.mid_theta[a] : 0.f, b < P.k ? P.mid_theta[b] : 0.f,
                                  a < P.k ? shift : -INFINITY, b < P.k ? shift : -INFINITY);
  }
  for (int j = tid; j < kMaxKpadTC / 4; j += kThreads) {
    auto val = [&](int kk, int pp) { return (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f; };
    auto mid = [&](int kk) { return kk < P.k ? P.mid_theta[kk] : 0.f; };
    const int a = 4 * j;
    S.yq[0][j] = make_float4(val(a, 0), val(a + 1, 0), val(a + 2, 0), val(a + 3, 0));
    S.yq[1][j] = make_float4(val(a, 1), val(a + 1, 1), val(a + 2, 1), val(a + 3, 1));
    S.yq[2][j] = make_float4(mid(a), mid(a + 1), mid(a + 2), mid(a + 3));
  }
  for (int j = tid; j < kMaxKpadTC + 8; j += kThreads) S.red[j] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.a_full[b], kBuildWarps);
      tc::mbar_init(&S.a_empty[b], kAccThreads / 32);
    }
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.b_full[s], kLoadThreads);
      tc::mbar_init(&S.b_empty[s], 1);
    }
    tc::mbar_init(&S.r_full, 1);
    tc::mbar_init(&S.r_empty, kAccThreads / 32);
  }
  if (warp == kAccWarp0) tc::tmem_alloc(&S.tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;

  if (warp < kMmaWarp || (warp > kMmaWarp && warp < kBuildWarp0)) {
    // ================= loaders: tap rows (D / 64 chunks), then G rows (2 chunks) =================
    reg_dealloc<kRegProducer>();
    const int lt = warp < kMmaWarp ? tid : tid - 32;  // loader thread index
    const int q = lt & 7, r0 = lt >> 3;
    int stage = 0;
    uint32_t phase = 0, il = 0;
    int4 e_nx = item_at(P, nwork, 0);
    for (int k = 0;; ++k) {
      const int4 e = e_nx;
      if (e.x >= 0) e_nx = item_at(P, nwork, k + 1);  // the next item's entry, loaded during this one
      if (e.x < 0) break;
      const int kt = e_kt(e), ktp = (kt + 15) & ~15;
      PF_DCHECK(kt > 0 && ktp <= kKt && e.y >= 0 && (int64_t)e.y + e_rows(e) <= ((P.n + P.tr - 1) / P.tr) * P.tr, "work item");
      int32_t* cell = S.cell[il & 1];
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      for (int v = lt; v < P.nv; v += kLoadThreads) {
        const uint2 ds = P.tile_desc[(int64_t)e.x * P.nv + v];
        const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
        const int ww = ds.y & 0xff, hh = (ds.y >> 8) & 0xff;
        const ViewF& vw = S.sv[v];
        const int sz = (ww * hh + 1) & ~1;  // padding tap: a valid row (zero weight)
        PF_DCHECK(sz == 0 || (base + sz <= ktp && x0 + ww <= vw.Wf && y0 + hh <= vw.Hf), "window inside the item / map");
        for (int a = 0; a < sz; ++a) {
          const int aa = a < ww * hh ? a : 0;
          cell[base + a] = vw.cell_base + (y0 + aa / ww) * vw.Wf + x0 + aa % ww;
        }
      }
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      int rc[kRowsPer];
#pragma unroll
      for (int j = 0; j < kRowsPer; ++j) {
        const int r = r0 + kRowStep * j;
        rc[j] = r < ktp ? cell[r < kt ? r : 0] : -1;  // rows kt..ktp-1 repeat tap 0 (finite, zero weight)
        PF_DCHECK(rc[j] < 0 || rc[j] < S.sv[P.nv - 1].cell_base + S.sv[P.nv - 1].Hf * S.sv[P.nv - 1].Wf, "tap row inside the maps");
      }
      for (int c = 0; c < nd + 2; ++c) {
        if constexpr (PROF) {
          const long long t0_ = clock64();
          GWAIT_SLEEP(&S.b_empty[stage], phase ^ 1u, PF_GRAM_SLEEP_NS);
          wcyc[0] += clock64() - t0_;
        } else {
          GWAIT_SLEEP(&S.b_empty[stage], phase ^ 1u, PF_GRAM_SLEEP_NS);  // loaders run ahead: sleep
        }
        const uint32_t sb = tc::smem_u32(sB + stage * kStageBytes);
        const uint16_t* src;
        int rowlen;
        if (c < nd) {
          src = reinterpret_cast<const uint16_t*>(P.fmap) + c * 64 + q * 8;
          rowlen = P.d;
        } else {
          src = P.Gbf + (c - nd) * 64 + q * 8;
          rowlen = P.kpadg;
        }
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j) {
          const int r = r0 + kRowStep * j;  // swizzled 16-byte piece q of row r
          if (rc[j] >= 0)
            tc::cp_async16(sb + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((q ^ r) & 7) << 4)),
                           src + (int64_t)rc[j] * rowlen);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&S.b_full[stage]))
                     : "memory");
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      }
      ++il;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    reg_dealloc<kRegProducer>();
    int stage = 0;
    uint32_t phase = 0, ruse = 0, wuse = 0;
    const uint32_t idS = tc::idesc_bf16_f32(128, kMaxKpadTC, false, true);
    const uint32_t mt0 = tc::smem_u32(sM);
    int4 e_nx = item_at(P, nwork, 0);
    for (int k = 0;; ++k) {
      const int4 e = e_nx;
      if (e.x >= 0) e_nx = item_at(P, nwork, k + 1);  // the next item's entry, loaded during this one
      if (e.x < 0) break;
      const int ktp = (e_kt(e) + 15) & ~15, nb = e_nb(e);
      // ---- Gram: block 0 = taps 0..127 x all, block 1 = taps 128.. x taps 128.. ----
      const uint32_t idG0 = tc::idesc_bf16_f32(128, ktp, false, false);
      const bool two = ktp > 128;
      const uint32_t idG1 = tc::idesc_bf16_f32(128, two ? ktp - 128 : 16, false, false);
      GWAITP(&S.r_empty, (ruse & 1u) ^ 1u, 1);
      for (int c = 0; c < nd; ++c) {
        GWAITP(&S.b_full[stage], phase, 2);
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(sB + stage * kStageBytes);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint64_t d0 = tc::smem_desc_sw128(a0 + s * 32, 16, 1024);
          tc::mma_bf16_ss_elect(tbase + kColG0, d0, d0, idG0, (c | s) ? 1u : 0u);
          if (two) {
            const uint64_t d1 = tc::smem_desc_sw128(a0 + 16384 + s * 32, 16, 1024);
            tc::mma_bf16_ss_elect(tbase + kColG1, d1, d1, idG1, (c | s) ? 1u : 0u);
          }
        }
        tc::mma_commit_elect(&S.b_empty[stage]);
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      }
      tc::mma_commit_elect(&S.r_full);
      ++ruse;
      // ---- per row block: S_b = W_b G_taps, Y_b = W_b M~ ----
      const int gs = stage;  // G chunk pair (adjacent stages, same phase)
      GWAITP(&S.b_full[gs], phase, 3);
      GWAITP(&S.b_full[gs + 1], phase, 3);
      // Y over N = ktp rounded up to 32 columns: M~ rows ktp.. are zero (the drain writes them), so the
      // accumulators read whole 32-column chunks without a bound check
      const uint32_t idY = tc::idesc_bf16_f32(128, (ktp + 31) & ~31, false, false);
      for (int b = 0; b < nb; ++b) {
        const int ab = (int)(wuse & 1u);
        GWAITP(&S.a_full[ab], (wuse >> 1) & 1u, 4);
        GWAITP(&S.r_empty, (ruse & 1u) ^ 1u, 5);  // Gram drained into M~ / previous block read
        tc::fence_after_sync();
        const uint32_t tA = tbase + kColW + (uint32_t)ab * kWCols;
        uint64_t bd = tc::smem_desc_sw128(tc::smem_u32(sB + gs * kStageBytes), kStageBytes, 1024);
        for (int s = 0; s < ktp / 16; ++s) {
          tc::mma_bf16_ts_elect(tbase + kColS, tA + 8u * s, bd, idS, s ? 1u : 0u);
          bd += 128;  // 16 rows x 128 B
        }
        for (int s = 0; s < ktp / 16; ++s) {
          const uint64_t md = tc::smem_desc_sw128(mt0 + (uint32_t)((s >> 2) * kChunkBytes + (s & 3) * 32), 16, 1024);
          tc::mma_bf16_ts_elect(tbase + kColY, tA + 8u * s, md, idY, s ? 1u : 0u);
        }
        tc::mma_commit_elect(&S.r_full);
        ++ruse;
        ++wuse;
      }
      tc::mma_commit_elect(&S.b_empty[gs]);
      tc::mma_commit_elect(&S.b_empty[gs + 1]);
      stage += 2;
      if (stage == kStages) { stage = 0; phase ^= 1u; }
    }
  } else if (warp < kAccWarp0) {
    // ================= builders: W_b straight into TMEM, per 128-row block =================
    // Builder warp 4 + j owns TMEM lane quarter bq = warp & 3 (rows 32 bq .. of each block) and the
    // views of rank = bh (mod 3), bh = j >> 2, among the item's views with taps. For each of its
    // views it writes all 32 rows' columns of the view's window (zeros where a row does not see the
    // view), so every A column is written exactly once. No barriers between builder warps: each
    // warp keeps its view list (per item) and expansion coefficients (per block) in its own slice of
    // shared memory. Taps: first-order expansion of fu, fv (fusion.py:83-86) around the centre of the
    // warp's 32 points, clamped into the item's window; 32-row groups wider than 2 kAffineR use the
    // exact fp32 projection, bit-identical to prep's (pf_tile_dev.cuh).
    reg_dealloc<kRegProducer>();
    const int bj = warp - kBuildWarp0, bq = warp & 3, bh = bj >> 2;
    const int row = 32 * bq + lane;
    const uint32_t t_lanes = (uint32_t)(32 * bq) << 16;
    const float wf1 = (float)(S.sv[0].Wf - 1), hf1 = (float)(S.sv[0].Hf - 1);
    const uint32_t below = (1u << lane) - 1u;
    int4* wl = S.wlist[bj];     // this warp's views: {view, window base | shape << 16, x0 | y0 << 8 | w << 16 | h << 24, -}
    float4* wc = S.wcoef[bj];   // and their expansion coefficients {A0, A1} for the current block
    uint32_t wuse = 0;
    int4 e_nx = item_at(P, nwork, 0);
    for (int k = 0;; ++k) {
      const int4 e = e_nx;
      if (e.x >= 0) e_nx = item_at(P, nwork, k + 1);  // the next item's entry, loaded during this one
      if (e.x < 0) break;
      PT(23);
      // this item's windows: views lane and lane + 32
      const uint2 d0 = lane < P.nv ? ld_pref_u2(P.tile_desc + (int64_t)e.x * P.nv + lane) : make_uint2(0u, 0u);
      const uint2 d1 = lane + 32 < P.nv ? ld_pref_u2(P.tile_desc + (int64_t)e.x * P.nv + lane + 32) : make_uint2(0u, 0u);
      const int kt = e_kt(e), ktp = (kt + 15) & ~15, nb = e_nb(e), nrows = e_rows(e);
      float4 p_nx = make_float4(0.f, 0.f, 0.f, 0.f);
      uint2 mw_nx = make_uint2(0u, 0u);
      if (row < nrows && (int64_t)e.y + row < P.n) {
        p_nx = ld_pref_f4(P.spts + e.y + row);
        mw_nx = ld_pref_u2(P.srec + e.y + row);
      }
      int nmine, n22, ncls[5];
      {  // this warp's views (rank = bh mod 3): the 2 x 2 windows first (built in pairs), then the rest
        const int c0 = shape_cls(d0), c1 = shape_cls(d1);
        const uint32_t m0 = __ballot_sync(0xffffffffu, c0 >= 0), m1 = __ballot_sync(0xffffffffu, c1 >= 0);
        const bool mine0 = c0 >= 0 && (int)(__popc(m0 & below) % kBuildGroups) == bh;
        const bool mine1 = c1 >= 0 && (int)((__popc(m0) + __popc(m1 & below)) % kBuildGroups) == bh;
        // order: 2 x 2, 3 x 2, 2 x 3, 3 x 3, other (classes 0..4); n_c views per class
        int pos0 = 0, pos1 = 0, tot = 0;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          const uint32_t a0 = __ballot_sync(0xffffffffu, mine0 && c0 == c), a1 = __ballot_sync(0xffffffffu, mine1 && c1 == c);
          if (c0 == c) pos0 = tot + __popc(a0 & below);
          if (c1 == c) pos1 = tot + __popc(a0) + __popc(a1 & below);
          ncls[c] = __popc(a0) + __popc(a1);
          tot += ncls[c];
        }
        n22 = ncls[0];
        nmine = tot;
        auto put = [&](int k, int v, uint2 d, int c) {
          PF_DCHECK((int)(d.x & 0xffff) + (((int)(d.y & 0xff) * (int)((d.y >> 8) & 0xff) + 1) & ~1) <= ktp &&
                        k < kMaxViewsTC / kBuildGroups + 1,
                    "builder window slot");
          wl[k] = make_int4(v, (int)(d.x & 0xffff) | (c << 16), (int)((d.x >> 16) & 0xffff) | (int)((d.y & 0xffff) << 16), 0);
        };
        if (mine0) put(pos0, lane, d0, c0);
        if (mine1) put(pos1, lane + 32, d1, c1);
        __syncwarp();
      }
      // expansion centre: the item's box, the union of the boxes prep recorded for its 128-row tiles
      // (a superset of its rows' box); the coefficients then serve every 128-row block of the item
      float ox = 0.f, oy = 0.f, oz = 0.f;
      bool exact;
      {
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        const int64_t t0 = (int64_t)e.y / kTile, t1 = ((int64_t)e.y + nrows - 1) / kTile;
        for (int64_t t = t0; t <= t1; ++t) {
          const float4 a = ld_pref_f4(P.tbox + 2 * t), c = ld_pref_f4(P.tbox + 2 * t + 1);
          lo[0] = fminf(lo[0], a.x);
          lo[1] = fminf(lo[1], a.y);
          lo[2] = fminf(lo[2], a.z);
          hi[0] = fmaxf(hi[0], c.x);
          hi[1] = fmaxf(hi[1], c.y);
          hi[2] = fmaxf(hi[2], c.z);
        }
        const bool any = lo[0] <= hi[0];
        if (any) {
          ox = 0.5f * (lo[0] + hi[0]);
          oy = 0.5f * (lo[1] + hi[1]);
          oz = 0.5f * (lo[2] + hi[2]);
        }
        const float ex = any ? hi[0] - lo[0] : 0.f, ey = any ? hi[1] - lo[1] : 0.f, ez = any ? hi[2] - lo[2] : 0.f;
        exact = ex * ex + ey * ey + ez * ez > 4.f * kAffineR * kAffineR;
      }
      if (!exact && lane < nmine) {  // lane k: coefficients of the warp's k-th view (relative to its window origin)
        const int4 wk = wl[lane];
        const float4* vp = S.vpk[wk.x];
        const float4 q0 = vp[0], q1 = vp[1], q2 = vp[2], kk = vp[3], mm = vp[4];
        const float X = fmaf(q0.z, oz, fmaf(q0.y, oy, q0.x * ox)) + q0.w;
        const float Y = fmaf(q1.z, oz, fmaf(q1.y, oy, q1.x * ox)) + q1.w;
        const float Z = fmaf(q2.z, oz, fmaf(q2.y, oy, q2.x * ox)) + q2.w;
        const float rz = __frcp_rn(Z), xr = X * rz, yr = Y * rz;  // (a first-order model: no IEEE division)
        const float su = mm.x * kk.x * rz, sv = mm.y * kk.z * rz;  // d fu / d X_cam, d fv / d Y_cam
        wc[2 * lane] = make_float4((fmaf(kk.x, xr, kk.y) + 0.5f) * mm.x - 0.5f - (float)(wk.z & 0xff),
                                   su * (q0.x - xr * q2.x), su * (q0.y - xr * q2.y), su * (q0.z - xr * q2.z));
        wc[2 * lane + 1] = make_float4((fmaf(kk.z, yr, kk.w) + 0.5f) * mm.y - 0.5f - (float)((wk.z >> 8) & 0xff),
                                       sv * (q1.x - yr * q2.x), sv * (q1.y - yr * q2.y), sv * (q1.z - yr * q2.z));
      }
      __syncwarp();
      PT(12);
      for (int b = 0; b < nb; ++b) {
        const float4 p = p_nx;
        const uint2 mw = mw_nx;
        const bool rv = 128 * b + row < nrows && (int64_t)e.y + 128 * b + row < P.n;
        if (b + 1 < nb) {  // next block's point and visibility word
          const int64_t jr = (int64_t)e.y + 128 * (b + 1) + row;
          p_nx = make_float4(0.f, 0.f, 0.f, 0.f);
          mw_nx = make_uint2(0u, 0u);
          if (128 * (b + 1) + row < nrows && jr < P.n) {
            p_nx = ld_pref_f4(P.spts + jr);
            mw_nx = ld_pref_u2(P.srec + jr);
          }
        }
        const int ab = (int)(wuse & 1u);
        const float dxp = p.x - ox, dyp = p.y - oy, dzp = p.z - oz;
        __syncwarp();
        PT(13);
        GWAITP(&S.a_empty[ab], ((wuse >> 1) & 1u) ^ 1u, 6);
        tc::fence_after_sync();
        PT(14);
        const uint32_t tAb = tbase + kColW + (uint32_t)ab * kWCols + t_lanes;
        // timing experiment (PF_GRAM_ABLATE & 4): weights computed but not stored to TMEM
        const bool nost = (P.ablate & 4) != 0;
        const int nunits = (P.ablate & 1) ? 0 : nmine;
        int k0 = 0;
        if (!exact && nunits) {
          // 2 x 2 windows, two views per step (independent chains): fu_rel, fv_rel in [0, 1] after the
          // clamp; weights (1-x)(1-y), x(1-y), (1-x)y, xy (numpy_impl.py:50-57) as two bf16 pairs
          auto w22 = [&](int k, uint32_t& lo, uint32_t& hi, uint32_t& col) {
            const int2 wk = *reinterpret_cast<const int2*>(&wl[k]);
            const float4 A0 = wc[2 * k], A1 = wc[2 * k + 1];
            const float wx = __saturatef(fmaf(A0.w, dzp, fmaf(A0.z, dyp, fmaf(A0.y, dxp, A0.x))));
            const float wy = __saturatef(fmaf(A1.w, dzp, fmaf(A1.z, dyp, fmaf(A1.y, dxp, A1.x))));
            const int v = wk.x;
            const float gg = (((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) ? 1.f : 0.f;
            const float ux = 1.f - wx, uy = gg - gg * wy, vy = gg * wy;
            lo = pack_bf16(uy * ux, uy * wx);
            hi = pack_bf16(vy * ux, vy * wx);
            col = tAb + (uint32_t)((wk.y & 0xffff) >> 1);
          };
          for (; k0 + 1 < n22; k0 += 2) {
            uint32_t l1, h1, c1, l2, h2, c2;
            w22(k0, l1, h1, c1);
            w22(k0 + 1, l2, h2, c2);
            if (nost) {
              asm volatile("" ::"r"(l1), "r"(h1), "r"(l2), "r"(h2));
            } else {
              tc::tmem_st_x2(c1, l1, h1);
              tc::tmem_st_x2(c2, l2, h2);
            }
          }
          if (k0 < n22) {
            uint32_t l1, h1, c1;
            w22(k0, l1, h1, c1);
            if (nost) asm volatile("" ::"r"(l1), "r"(h1)); else tc::tmem_st_x2(c1, l1, h1);
            ++k0;
          }
          // 3 x 2 and 2 x 3 windows in pairs: separable weights over the 3-tap side (vx0, vx1, vx2) and
          // the 2-tap side; three bf16 pairs each (taps in row-major window order)
          auto w3 = [&](int k, bool wide, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& col) {
            const int2 wk = *reinterpret_cast<const int2*>(&wl[k]);
            const float4 A0 = wc[2 * k], A1 = wc[2 * k + 1];
            const float fu = fmaf(A0.w, dzp, fmaf(A0.z, dyp, fmaf(A0.y, dxp, A0.x)));
            const float fv = fmaf(A1.w, dzp, fmaf(A1.z, dyp, fmaf(A1.y, dxp, A1.x)));
            const int v = wk.x;
            const float gg = (((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) ? 1.f : 0.f;
            // the 3-tap side: t in [0, 2], cell i = min(floor(t), 1), weight t - i
            const float t3 = fminf(fmaxf(wide ? fu : fv, 0.f), 2.f), t2 = __saturatef(wide ? fv : fu);
            const float i3 = fminf(floorf(t3), 1.f), f3 = t3 - i3;
            const bool lo3 = i3 == 0.f;
            const float s0 = lo3 ? 1.f - f3 : 0.f, s1 = lo3 ? f3 : 1.f - f3, s2 = lo3 ? 0.f : f3;
            const float q0 = gg - gg * t2, q1 = gg * t2;  // the 2-tap side
            if (wide) {  // 3 x 2: r0 = (s0 s1 s2) q0, r1 = (s0 s1 s2) q1
              a = pack_bf16(q0 * s0, q0 * s1);
              b = pack_bf16(q0 * s2, q1 * s0);
              c = pack_bf16(q1 * s1, q1 * s2);
            } else {  // 2 x 3: rows s0, s1, s2 of (q0 q1) (q: the x side here)
              a = pack_bf16(s0 * q0, s0 * q1);
              b = pack_bf16(s1 * q0, s1 * q1);
              c = pack_bf16(s2 * q0, s2 * q1);
            }
            col = tAb + (uint32_t)((wk.y & 0xffff) >> 1);
          };
          auto st3 = [&](uint32_t col, uint32_t a, uint32_t b, uint32_t c) {
            if (nost) {
              asm volatile("" ::"r"(a), "r"(b), "r"(c));
            } else {
              tc::tmem_st_x2(col, a, b);
              tc::tmem_st_x1(col + 2u, c);
            }
          };
          for (int cl = 1; cl <= 2; ++cl) {
            const int kend = k0 + ncls[cl];
            const bool wide = cl == 1;
            for (; k0 + 1 < kend; k0 += 2) {
              uint32_t a1, b1, c1, col1, a2, b2, c2, col2;
              w3(k0, wide, a1, b1, c1, col1);
              w3(k0 + 1, wide, a2, b2, c2, col2);
              st3(col1, a1, b1, c1);
              st3(col2, a2, b2, c2);
            }
            if (k0 < kend) {
              uint32_t a1, b1, c1, col1;
              w3(k0, wide, a1, b1, c1, col1);
              st3(col1, a1, b1, c1);
              ++k0;
            }
          }
        }
        for (int k = k0; k < nunits; ++k) {  // warp-uniform: one view (32 rows) per iteration
          const int4 wk = wl[k];
          const int v = wk.x, base = wk.y & 0xffff, cls = wk.y >> 16;
          float fu_rel, fv_rel;
          if (!exact) {
            const float4 A0 = wc[2 * k], A1 = wc[2 * k + 1];
            fu_rel = fmaf(A0.w, dzp, fmaf(A0.z, dyp, fmaf(A0.y, dxp, A0.x)));
            fv_rel = fmaf(A1.w, dzp, fmaf(A1.z, dyp, fmaf(A1.y, dxp, A1.x)));
          } else {
            const ProjF pr = project_f32(S.sv[v], p.x, p.y, p.z);
            const TapF tf = taps_f32(S.sv[v], pr.u, pr.v);
            fu_rel = (float)(tf.x0 - (wk.z & 0xff)) + tf.wx;
            fv_rel = (float)(tf.y0 - ((wk.z >> 8) & 0xff)) + tf.wy;
          }
          const float gg = ((((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) != 0u) ? 1.f : 0.f;
          const uint32_t col = tAb + (uint32_t)(base >> 1);
          if (cls == 0) {  // 2 x 2 (most windows): fu_rel, fv_rel in [0, 1] after the clamp
            const float wx = __saturatef(fu_rel), wy = __saturatef(fv_rel);
            const float ux = 1.f - wx, uy = gg - gg * wy, vy = gg * wy;
            const uint32_t a = pack_bf16(uy * ux, uy * wx), c = pack_bf16(vy * ux, vy * wx);
            if (nost) asm volatile("" ::"r"(a), "r"(c)); else tc::tmem_st_x2(col, a, c);
          } else if (cls <= 3) {  // sides 2 or 3: separable weights; the clamp reproduces the reference taps
            const int ww = cls == 2 ? 2 : 3, wh = cls == 1 ? 2 : 3;
            const float xr = fminf(fmaxf(fu_rel, 0.f), (float)(ww - 1)), yr = fminf(fmaxf(fv_rel, 0.f), (float)(wh - 1));
            const float ixf = fminf(floorf(xr), (float)(ww - 2)), iyf = fminf(floorf(yr), (float)(wh - 2));
            const float wx = xr - ixf, wy = yr - iyf;
            const bool xa = ixf == 0.f, ya = iyf == 0.f;
            const float vx0 = xa ? 1.f - wx : 0.f, vx1 = xa ? wx : 1.f - wx, vx2 = xa ? 0.f : wx;
            const float vy0 = ya ? gg * (1.f - wy) : 0.f, vy1 = ya ? gg * wy : gg * (1.f - wy), vy2 = ya ? 0.f : gg * wy;
            if (cls == 1) {  // 3 x 2: taps r0: 0 1 2, r1: 3 4 5
              const uint32_t a = pack_bf16(vy0 * vx0, vy0 * vx1), c = pack_bf16(vy0 * vx2, vy1 * vx0),
                             d = pack_bf16(vy1 * vx1, vy1 * vx2);
              if (nost) asm volatile("" ::"r"(a), "r"(c), "r"(d));
              else {
                tc::tmem_st_x2(col, a, c);
                tc::tmem_st_x1(col + 2u, d);
              }
            } else if (cls == 2) {  // 2 x 3: taps r0: 0 1, r1: 2 3, r2: 4 5
              const uint32_t a = pack_bf16(vy0 * vx0, vy0 * vx1), c = pack_bf16(vy1 * vx0, vy1 * vx1),
                             d = pack_bf16(vy2 * vx0, vy2 * vx1);
              if (nost) asm volatile("" ::"r"(a), "r"(c), "r"(d));
              else {
                tc::tmem_st_x2(col, a, c);
                tc::tmem_st_x1(col + 2u, d);
              }
            } else {  // 3 x 3: taps 0..8 + one padding tap
              const uint32_t a = pack_bf16(vy0 * vx0, vy0 * vx1), c = pack_bf16(vy0 * vx2, vy1 * vx0),
                             d = pack_bf16(vy1 * vx1, vy1 * vx2), f = pack_bf16(vy2 * vx0, vy2 * vx1),
                             g = pack_bf16(vy2 * vx2, 0.f);
              if (nost) asm volatile("" ::"r"(a), "r"(c), "r"(d), "r"(f), "r"(g));
              else {
                tc::tmem_st_x4(col, a, c, d, f);
                tc::tmem_st_x1(col + 4u, g);
              }
            }
          } else {  // other window shapes: the general bilinear rule (numpy_impl.py:50-57) inside the window
            const int wx0 = wk.z & 0xff, wy0 = (wk.z >> 8) & 0xff, ww = (wk.z >> 16) & 0xff, wh = (wk.z >> 24) & 0xff;
            const float fu = fu_rel + (float)wx0, fv = fv_rel + (float)wy0;
            const float x = fminf(fmaxf(fu, 0.f), wf1), y = fminf(fmaxf(fv, 0.f), hf1);
            const float xf = floorf(x), yf = floorf(y);
            float wx = x - xf, wy = y - yf;
            int ix = (int)xf - wx0, iy = (int)yf - wy0;
            bool dxb = xf < wf1, dyb = yf < hf1;
            if (ix < 0) { ix = 0; wx = 0.f; }
            if (ix > ww - 1) { ix = ww - 1; dxb = false; }
            if (ix + 1 > ww - 1) dxb = false;
            if (iy < 0) { iy = 0; wy = 0.f; }
            if (iy > wh - 1) { iy = wh - 1; dyb = false; }
            if (iy + 1 > wh - 1) dyb = false;
            float w00 = (1.f - wy) * (1.f - wx), w01 = (1.f - wy) * wx;
            float w10 = wy * (1.f - wx), w11 = wy * wx;
            if (!dxb) { w00 += w01; w10 += w11; }
            if (!dyb) { w00 += w10; w01 += w11; }
            const int t00 = iy * ww + ix;
            const int t01 = dxb ? t00 + 1 : -1, t10 = dyb ? t00 + ww : -1, t11 = (dxb && dyb) ? t00 + ww + 1 : -1;
            auto tapw = [&](int k2) {
              return gg * ((k2 == t00 ? w00 : 0.f) + (k2 == t01 ? w01 : 0.f) + (k2 == t10 ? w10 : 0.f) +
                           (k2 == t11 ? w11 : 0.f));
            };
            const int ncols = (ww * wh + 1) >> 1;
            for (int j = 0; j < ncols; ++j) {
              const uint32_t a = pack_bf16(tapw(2 * j), tapw(2 * j + 1));
              if (nost) asm volatile("" ::"r"(a)); else tc::tmem_st_x1(col + (uint32_t)j, a);
            }
          }
        }
        if (bh == 0)  // K padding columns (kt .. ktp) and the |F|^2 chunk tail (.. ktp rounded to 32) are zero
          for (int j = kt >> 1; j < (((ktp + 31) & ~31) >> 1); ++j) tc::tmem_st_x1(tAb + (uint32_t)j, 0u);
        PT(15);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.a_full[ab]);
        PT(16);
        ++wuse;
      }
    }
  } else {
    // ================= accumulators =================
    reg_alloc<kRegAcc>();
    const int half = (warp - kAccWarp0) >> 2;
    const int qd = warp & 3;
    const int row = 32 * qd + lane;
    const uint32_t t_lane = (uint32_t)(32 * qd) << 16;
    const int k0 = half * kHalfK;
    uint32_t ruse = 0, wuse = 0;
    float wsum[kHalfK / 32];
#pragma unroll
    for (int q = 0; q < kHalfK / 32; ++q) wsum[q] = 0.f;
    float pm_sum = 0.f, pmx = 0.f, pmy = 0.f, pmz = 0.f, featured_n = 0.f, pairs = 0.f;
    const bool p_wide = P.p > 2;
    int4 e_nx = item_at(P, nwork, 0);
    for (int k = 0;; ++k) {
      const int4 e = e_nx;
      if (e.x >= 0) e_nx = item_at(P, nwork, k + 1);  // the next item's entry, loaded during this one
      if (e.x < 0) break;
      const int ktp = (e_kt(e) + 15) & ~15, nb = e_nb(e), nrows = e_rows(e);
      uint2 rec_nx = make_uint2(0u, 0u);
      float4 pc_nx = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < nrows && (int64_t)e.y + row < P.n) {
        rec_nx = ld_pref_u2(reinterpret_cast<const uint32_t*>(P.srec + e.y + row) + 2);
        pc_nx = ld_pref_f4(P.spts + e.y + row);
      }
      PT(22);
      {
        // ---- Gram -> M~ (bf16, K-major SW128 rows of taps) ----
        GWAITP(&S.r_full, ruse & 1u, 7);
        ++ruse;
        tc::fence_after_sync();
        const bool two = ktp > 128;
        for (int j = half; j < 3; j += 2) {  // block 0, K chunk j (columns 64 j ..)
          if (64 * j >= ktp) continue;
          float v[64];
          tc::tmem_ld64(tbase + kColG0 + 64u * j + t_lane, v);
          if (row < ktp) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint4 u4 = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                          pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
              *reinterpret_cast<uint4*>(sM + mt_off(row, j, q)) = u4;
            }
            if (j == 2) {  // M[row][128 + m] -> M~ row 128 + m, column row (symmetric)
              const int jc = row >> 6, qc = (row & 63) >> 3, ec = row & 7;
#pragma unroll
              for (int m = 0; m < 64; ++m)
                if (128 + m < ktp) {
                  const int n = 128 + m;
                  *reinterpret_cast<__nv_bfloat16*>(sM + mt_off(n, jc, qc) + 2 * ec) = __float2bfloat16_rn(v[m]);
                }
            }
          }
        }
        {  // zero rows ktp .. ktp rounded to 32 (Y's N padding): <= 16 rows x the K chunks below ktp
          const int t = row + 128 * half, n = ktp + (t & 15), j = t >> 4;
          if (j < 3 && 64 * j < ktp && n < ((ktp + 31) & ~31))
#pragma unroll
            for (int q = 0; q < 8; ++q) *reinterpret_cast<uint4*>(sM + mt_off(n, j, q)) = make_uint4(0u, 0u, 0u, 0u);
        }
        if (two && half == 1) {  // block 1: rows 128 + row, columns 128..
          float v[64];
          tc::tmem_ld64(tbase + kColG1 + t_lane, v);
          if (128 + row < ktp) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint4 u4 = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                          pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
              *reinterpret_cast<uint4*>(sM + mt_off(128 + row, 2, q)) = u4;
            }
          }
        }
        tc::fence_async_shared();  // generic st.shared -> visible to the MMA (async proxy)
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.r_empty);
        PT(17);
      }
      for (int b = 0; b < nb; ++b) {
        // ---- row block ----
        const uint2 rec = rec_nx;
        const float4 pcur = pc_nx;
        const int rb = 128 * b + row;
        const int64_t jpt = (int64_t)e.y + rb;
        const bool valid = rb < nrows && jpt < P.n;
        if (b + 1 < nb) {
          rec_nx = make_uint2(0u, 0u);
          pc_nx = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rb + 128 < nrows && jpt + 128 < P.n) {
            rec_nx = ld_pref_u2(reinterpret_cast<const uint32_t*>(P.srec + jpt + 128) + 2);
            pc_nx = ld_pref_f4(P.spts + jpt + 128);
          }
        }
        const int ab = (int)(wuse & 1u);
        const int bp = ab;  // exchange-slot parity of this block
        ++wuse;
        GWAITP(&S.r_full, ruse & 1u, 8);
        ++ruse;
        tc::fence_after_sync();
        // |F|^2 = sum_t W[row, t] Y[row, t]: this half takes 32-column chunks c = half, half + 2, ...
        float ss = 0.f;
        const uint32_t tW = tbase + kColW + (uint32_t)ab * kWCols + t_lane;
        {
          uint64_t ss2 = 0ull;
          for (int c = half; 32 * c < ktp; c += 2) {  // whole chunks: columns ktp.. are zero
            uint32_t y[32], wr[16];
            tmem_ld_yw(tbase + kColY + 32u * c + t_lane, tW + 16u * c, y, wr);
#pragma unroll
            for (int q = 0; q < 16; ++q)  // bf16 pair -> two floats (exact: bf16 is the top half)
              ss2 = ffma2(pk2(__uint_as_float(wr[q] << 16), __uint_as_float(wr[q] & 0xffff0000u)),
                          pk2(__uint_as_float(y[2 * q]), __uint_as_float(y[2 * q + 1])), ss2);
          }
          float s_a, s_b;
          up2(ss2, s_a, s_b);
          ss = s_a + s_b;
        }
        PT(18);
        float v[kHalfK];
        tc::tmem_ld64(tbase + kColS + (uint32_t)k0 + t_lane, v);
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&S.r_empty);     // S, Y are in registers
          mbar_arrive(&S.a_empty[ab]);  // W read
        }
        PT(19);
        if (P.ablate & 2) continue;
        S.xss[bp][half][row] = ss;
        acc_pair_sync(qd);
        PT(20);
        const float fss = S.xss[bp][0][row] + S.xss[bp][1][row];
        const int count = (int)rec.x;
        const bool featured = valid && count > 0;
        const float inv = fss > 0.f ? rsqrtf(fss) : 0.f;
        const float sc = inv * P.inv_temp * 1.4426950408889634f;
        const int32_t pi = valid ? __float_as_int(pcur.w) : 0;
        if (OUTS && P.sims && valid) {
#pragma unroll
          for (int q = 0; q < kHalfK; ++q)
            if (k0 + q < P.k) P.sims[(int64_t)pi * P.k + k0 + q] = featured ? v[q] * inv : 0.f;
        }
        float m2 = 0.f;
        if (need_max) {
          float mx = -INFINITY;
#pragma unroll
          for (int q = 0; q < kHalfK; ++q) {
            const float4 yb = S.yp[2 * ((k0 + q) >> 1) + 1];
            mx = fmaxf(mx, fmaf(v[q], sc, (q & 1) ? yb.w : yb.z));
          }
          S.xm[bp][half][row] = mx;
          acc_pair_sync(qd);
          m2 = fmaxf(S.xm[bp][0][row], S.xm[bp][1][row]);
          if (!(m2 > -INFINITY)) m2 = 0.f;
        }
        float se, pl0, pl1, pl2 = 0.f, pl3 = 0.f, pml;
        {
          uint64_t sep = 0ull, p0p = 0ull, p1p = 0ull, pmp = 0ull;
          const uint64_t scp = pk2(sc, sc);
          // exponents v sc + shift (- row max only when need_max: a separate copy of the loop)
          auto softmax_pass = [&](auto with_max) {
            constexpr bool kMax = decltype(with_max)::value;
#pragma unroll
            for (int q = 0; q < kHalfK; q += 2) {
              if ((q & 15) == 0) asm volatile("" ::: "memory");
              const int kp = (k0 + q) >> 1;
              const float4 ya = S.yp[2 * kp], yb = S.yp[2 * kp + 1];
              float x0, x1;
              up2(ffma2(pk2(v[q], v[q + 1]), scp, kMax ? pk2(yb.z - m2, yb.w - m2) : pk2(yb.z, yb.w)), x0, x1);
              const float e0 = ex2(x0), e1 = ex2(x1);
              const uint64_t ee = pk2(e0, e1);
              sep = fadd2(sep, ee);
              p0p = ffma2(ee, pk2(ya.x, ya.y), p0p);
              p1p = ffma2(ee, pk2(ya.z, ya.w), p1p);
              pmp = ffma2(ee, pk2(yb.x, yb.y), pmp);
              v[q] = e0;
              v[q + 1] = e1;
            }
          };
          // the common case (no row max, no padding materials in this half): 4 materials per step,
          // the uniform shift in a register and 3 coefficient loads per 4 materials instead of 4 (the
          // loop is bound by the shared-memory / special-function issue queue)
          auto softmax_pass4 = [&]() {
            const uint64_t shp = pk2(shift, shift);
#pragma unroll
            for (int q = 0; q < kHalfK; q += 4) {
              if ((q & 15) == 0) asm volatile("" ::: "memory");
              const int g = (k0 + q) >> 2;
              const float4 c0 = S.yq[0][g], c1 = S.yq[1][g], cm = S.yq[2][g];
              float x0, x1, x2, x3;
              up2(ffma2(pk2(v[q], v[q + 1]), scp, shp), x0, x1);
              up2(ffma2(pk2(v[q + 2], v[q + 3]), scp, shp), x2, x3);
              const float e0 = ex2(x0), e1 = ex2(x1), e2 = ex2(x2), e3 = ex2(x3);
              const uint64_t ea = pk2(e0, e1), eb = pk2(e2, e3);
              sep = fadd2(sep, ea);
              sep = fadd2(sep, eb);
              p0p = ffma2(ea, pk2(c0.x, c0.y), p0p);
              p0p = ffma2(eb, pk2(c0.z, c0.w), p0p);
              p1p = ffma2(ea, pk2(c1.x, c1.y), p1p);
              p1p = ffma2(eb, pk2(c1.z, c1.w), p1p);
              pmp = ffma2(ea, pk2(cm.x, cm.y), pmp);
              pmp = ffma2(eb, pk2(cm.z, cm.w), pmp);
              v[q] = e0;
              v[q + 1] = e1;
              v[q + 2] = e2;
              v[q + 3] = e3;
            }
          };
          if (need_max) softmax_pass(std::true_type{});
          else if (k0 + kHalfK > P.k) softmax_pass(std::false_type{});  // padding materials: -inf shifts
          else softmax_pass4();
          if (p_wide) {
#pragma unroll
            for (int q = 0; q < kHalfK; ++q) {
              if ((q & 7) == 0) asm volatile("" ::: "memory");
              const float2 y2 = S.yv2[k0 + q];
              pl2 = fmaf(v[q], y2.x, pl2);
              pl3 = fmaf(v[q], y2.y, pl3);
            }
          }
          float a, c;
          up2(sep, a, c);
          se = a + c;
          up2(p0p, a, c);
          pl0 = a + c;
          up2(p1p, a, c);
          pl1 = a + c;
          up2(pmp, a, c);
          pml = a + c;
        }
        S.xsum[bp][half][0][row] = se;
        S.xsum[bp][half][1][row] = pl0;
        S.xsum[bp][half][2][row] = pl1;
        S.xsum[bp][half][3][row] = pl2;
        S.xsum[bp][half][4][row] = pl3;
        S.xsum[bp][half][5][row] = pml;
        acc_pair_sync(qd);
        PT(21);
        const float se_t = S.xsum[bp][0][0][row] + S.xsum[bp][1][0][row];
        if (featured && !(se_t <= 3.4e38f)) atomicOr(P.status, isnan(se_t) ? 1 : 2);
        const float rs = featured ? 1.f / se_t : 0.f;
        {
          const uint64_t rsp = pk2(rs, rs);
#pragma unroll
          for (int q = 0; q < kHalfK; q += 2) up2(ffma2(pk2(v[q], v[q + 1]), rsp, 0ull), v[q], v[q + 1]);
        }
        if (OUTS && P.weights && valid) {
#pragma unroll
          for (int q = 0; q < kHalfK; ++q)
            if (k0 + q < P.k) P.weights[(int64_t)pi * P.k + k0 + q] = v[q];
        }
        static_assert(kHalfK == 64, "32 material pairs per half");
        {
          // weight totals over the warp's 32 rows: the 64 weights as 32 bf16 pairs, one packed
          // reduce-scatter (half the shuffles of two fp32 ones); lane l ends with materials 2l, 2l + 1.
          // bf16 keeps fp32's range (tiny weights survive), and its round-to-nearest errors (2^-9 per
          // add) are unbiased, so the per-material totals over all points stay far inside the 1e-2 bar
          uint32_t pw[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) pw[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
          const uint32_t r = warp_reduce_scatter32_bf16x2(pw, lane);
          wsum[0] += __uint_as_float(r << 16);
          wsum[1] += __uint_as_float(r & 0xffff0000u);
        }
        if (valid && half == 0) {
          float prop[4];
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) prop[pp] = (S.xsum[bp][0][1 + pp][row] + S.xsum[bp][1][1 + pp][row]) * rs;
          const float pm = (S.xsum[bp][0][5][row] + S.xsum[bp][1][5][row]) * rs;
          *(reinterpret_cast<float4*>(P.srec + jpt) + 1) = make_float4(prop[0], prop[1], prop[2], prop[3]);
          if (P.grid_partials && (int32_t)rec.y >= 0) {  // code -1: a padding slot
            const int32_t code = (int32_t)rec.y;
            const int dc = P.density_col;
            const float rho = dc == 0 ? prop[0] : (dc == 1 ? prop[1] : (dc == 2 ? prop[2] : prop[3]));
            atomicAdd(P.grid_partials + code, rho);
            atomicAdd(P.grid_partials + P.cells3 + code, 1.0f);
          }
          const bool live = (int32_t)rec.y >= 0;  // a padding slot (NaN point): no partial contribution
          pm_sum += live ? pm : 0.f;
          pmx = fmaf(live ? pm : 0.f, live ? pcur.x : 0.f, pmx);
          pmy = fmaf(live ? pm : 0.f, live ? pcur.y : 0.f, pmy);
          pmz = fmaf(live ? pm : 0.f, live ? pcur.z : 0.f, pmz);
          featured_n += featured ? 1.f : 0.f;
          pairs += (float)count;
        }
        // (no closing barrier: the next block writes the other parity's slots, and the block after
        // that only gets past the next block's barriers once every thread has read these)
        PT(22);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // materials k0 + 2 lane + q
      const int k = k0 + 2 * lane + q;
      if (k < P.k && wsum[q] != 0.f) atomicAdd(&S.red[k], (double)wsum[q]);
    }
    double r6[6] = {pm_sum, pmx, pmy, pmz, featured_n, pairs};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      double x = r6[q];
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) atomicAdd(&S.red[P.k + q], x);
    }
    asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
    for (int j = tid - kAccWarp0 * 32; j < P.k + 6; j += kAccThreads)
      if (S.red[j] != 0.0) atomicAdd(P.partials + j, S.red[j]);
  }
  if (PROF && P.dbg && lane == 0) {
    wcyc[11] = clock64() - t_start;
    unsigned long long* d = P.dbg + blockIdx.x * 32;
    if (warp == 0) atomicAdd(d + 0, (unsigned long long)wcyc[0]);
    if (warp == kMmaWarp)
      for (int q = 1; q <= 5; ++q) atomicAdd(d + q, (unsigned long long)wcyc[q]);
    if (warp == kBuildWarp0) {
      atomicAdd(d + 6, (unsigned long long)wcyc[6]);
      atomicAdd(d + 9, (unsigned long long)(wcyc[11] - wcyc[6]));
      for (int q = 12; q <= 16; ++q) atomicAdd(d + q, (unsigned long long)wcyc[q]);
      atomicAdd(d + 23, (unsigned long long)wcyc[23]);
    }
    if (warp == kAccWarp0) {
      atomicAdd(d + 7, (unsigned long long)wcyc[7]);
      atomicAdd(d + 8, (unsigned long long)wcyc[8]);
      atomicAdd(d + 10, (unsigned long long)(wcyc[11] - wcyc[7] - wcyc[8]));
      atomicAdd(d + 11, (unsigned long long)wcyc[11]);
      for (int q = 17; q <= 22; ++q) atomicAdd(d + q, (unsigned long long)wcyc[q]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kAccWarp0) tc::tmem_dealloc(tbase, 512);
  if (P.ctatime && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    P.ctatime[2 * blockIdx.x] = t_cta0;
    P.ctatime[2 * blockIdx.x + 1] = t1;
  }
#undef PT
}

// Work items -> the compact list the tile kernel walks (items that fit the tap budget) and the
// SIMT kernel's point list (rows of items with no visible taps, or more than kKt taps and not split
// further). One warp per 512-row tile (and its 128-row tiles when it overflows) or per 32-row item.
__global__ void k_collect_work(TileParams P) {
  const int64_t nt = (P.n + P.tr - 1) / P.tr;
  const int n2 = min(*P.sub2_count, P.max_sub2);
  const int64_t first2 = nt + 4 * (int64_t)P.max_sub_tiles;
  const int lane = threadIdx.x & 31;
  auto push = [&](int64_t item, int64_t row0, int rows, int kt) {
    if (lane != 0) return;
    const int4 e = make_int4((int)item, (int)row0, rows | (kt << 16), 0);
    // split items (128 / 32 rows: item ids >= nt) run in the feature-product kernel: per 128 rows the
    // Gram product (kt^2 D) costs more than the feature product (128 kt D) once kt exceeds ~128. (Not
    // by row count: the last 512-row tile of an object may be short but is still a 512-row item.)
    const int64_t cap = nt + 4 * (int64_t)P.max_sub_tiles + 4 * (int64_t)P.max_sub2;  // list capacity
    if (P.wlist && item >= nt) {
      const int slot = atomicAdd(P.wcount, 1);
      PF_DCHECK(slot < cap, "split-item list slot");
      P.wlist[slot] = e;
    } else {
      const int slot = atomicAdd(P.work_count, 1);
      PF_DCHECK(slot < cap, "work list slot");
      P.work_raw[slot] = e;
    }
  };
  auto overflow = [&](int64_t row0, int rows) {
    for (int r = lane; r < rows; r += 32) P.ovf_list[atomicAdd(P.ovf_count, 1)] = __float_as_int(P.spts[row0 + r].w);
  };
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nt + 4 * (int64_t)n2;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    bool ok;
    if (w < nt) {
      const int kt = P.tile_kt[w];
      const int rows = (int)min((int64_t)P.tr, P.n - w * P.tr);
      ktp_ok(kt, ok);
      if (ok) {
        push(w, w * P.tr, rows, kt);
      } else if (kt <= 0) {
        overflow(w * P.tr, rows);  // nothing visible: featureless points
      } else {
        for (int q = 0; q < P.tr / kTile; ++q) {  // the 128-row tiles (level-1 items)
          const int64_t r0 = w * P.tr + q * kTile;
          if (r0 >= P.n) break;
          const int k = P.tile_kt[nt + w * (P.tr / kTile) + q];
          const int r = (int)min((int64_t)kTile, P.n - r0);
          if (k == -1) continue;  // split into 32-row items
          ktp_ok(k, ok);
          if (ok) push(nt + w * (P.tr / kTile) + q, r0, r, k);
          else overflow(r0, r);
        }
      }
    } else {
      const int64_t u = w - nt;
      const int64_t item = first2 + u;
      const int64_t r0 = ((int64_t)P.sub2_items[u >> 2] - nt) * kTile + 32 * (u & 3);
      if (r0 >= P.n) continue;
      const int r = (int)min((int64_t)32, P.n - r0);
      const int k = P.tile_kt[item];
      ktp_ok(k, ok);
      if (ok) push(item, r0, r, k);
      else overflow(r0, r);
    }
  }
}

// The collected list (arbitrary order: atomics) -> P.work sorted by estimated cost, descending: a
// counting sort over 32 buckets of rows x taps in one CTA (C5: 32k items, a few microseconds).
__global__ void __launch_bounds__(1024) k_sort_work(TileParams P) {
  __shared__ int cnt[32];
  const int n = *P.work_count, tid = threadIdx.x, lane = tid & 31;
  auto key = [](const int4& e) { return 31 - min((e_nb(e) * e_kt(e)) >> 5, 31); };
  if (tid < 32) cnt[tid] = 0;
  __syncthreads();
  // warp-aggregated counts (most items of a warp share a bucket); the loop bound is warp-uniform.
  // Both passes load kU entries per thread before using any (one CTA: the loop is latency-bound)
  constexpr int kU = 4;
  for (int i0 = tid - lane; i0 < n; i0 += kU * blockDim.x) {
    int kk[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x + lane;
      kk[u] = i < n ? key(P.work_raw[i]) : -1;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t peers = __match_any_sync(0xffffffffu, kk[u]);
      if (kk[u] >= 0 && (peers & ((1u << lane) - 1u)) == 0u) atomicAdd(&cnt[kk[u]], __popc(peers));
    }
  }
  __syncthreads();
  if (tid < 32) {  // exclusive scan of the 32 bucket counts
    const int c = cnt[tid];
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (tid >= o) incl += t;
    }
    cnt[tid] = incl - c;
  }
  __syncthreads();
  for (int i0 = tid - lane; i0 < n; i0 += kU * blockDim.x) {
    int4 e[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x + lane;
      e[u] = i < n ? P.work_raw[i] : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = i0 + u * blockDim.x + lane;
      const int kk = i < n ? key(e[u]) : -1;
      const uint32_t peers = __match_any_sync(0xffffffffu, kk);
      const int leader = __ffs(peers) - 1;
      int base = 0;
      if (kk >= 0 && lane == leader) base = atomicAdd(&cnt[kk], __popc(peers));
      base = __shfl_sync(peers, base, leader);
      if (kk >= 0) P.work[base + __popc(peers & ((1u << lane) - 1u))] = e[u];
    }
  }
}

}  // namespace

int run_tile_gram(const TileParams& P, cudaStream_t st) {
  if (P.kpadg != kMaxKpadTC) return set_error(PF_ERR_VALUE, "tile_gram: S operand must be %d wide", kMaxKpadTC);
  if (P.x3) return set_error(PF_ERR_VALUE, "tile_gram: bf16 maps only");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)kStages * kStageBytes + kMtBytes + 1024;
  cudaFuncSetAttribute(k_tile_gram<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_gram<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_gram<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (P.n + P.tr - 1) / P.tr;
  int grid = sms;  // persistent: CTAs stride over the device-side work list (empty CTAs exit)
  if (const char* g = getenv("PF_WS_GRID")) grid = atoi(g) > 0 ? atoi(g) : grid;  // debug knob
  if (grid < 1) grid = 1;
  cudaMemsetAsync(P.work_count, 0, sizeof(int32_t), st);
  if (P.wlist) cudaMemsetAsync(P.wcount, 0, sizeof(int32_t), st);
  k_collect_work<<<grid_for(32 * (ntiles + 4 * (int64_t)P.max_sub2), 256, 148 * 8), 256, 0, st>>>(P);
  if (int rc = check_launch("collect_work")) return rc;
  k_sort_work<<<1, 1024, 0, st>>>(P);
  if (int rc = check_launch("sort_work")) return rc;
  const bool debug = getenv("PF_WS_DEBUG") != nullptr;
  static unsigned long long* dbg = nullptr;
  TileParams Q = P;
  static unsigned long long* ctat = nullptr;
  const bool ctatime = getenv("PF_GRAM_CTATIME") != nullptr;
  if (ctatime) {
    if (!ctat) cudaMalloc(&ctat, sizeof(unsigned long long) * 2 * 1024);
    Q.ctatime = ctat;
  }
  if (const char* ab = getenv("PF_GRAM_ABLATE")) Q.ablate = atoi(ab);
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 32 * 1024);
    cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 32 * 1024, st);
    Q.dbg = dbg;
    k_tile_gram<false, true><<<grid, kThreads, smem, st>>>(Q);
  } else if (P.sims || P.weights) {
    k_tile_gram<true, false><<<grid, kThreads, smem, st>>>(Q);
  } else {
    k_tile_gram<false, false><<<grid, kThreads, smem, st>>>(Q);
  }
  int rc = check_launch("tile_gram");
  if (ctatime && rc == PF_OK) {  // CTA time spread of this launch (production instantiation)
    static unsigned long long h[2 * 1024];
    cudaMemcpyAsync(h, ctat, sizeof(unsigned long long) * 2 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long s0 = ~0ull, e1 = 0, e0 = ~0ull;
    double mean = 0;
    for (int b = 0; b < grid; ++b) {
      s0 = h[2 * b] < s0 ? h[2 * b] : s0;
      e1 = h[2 * b + 1] > e1 ? h[2 * b + 1] : e1;
      e0 = h[2 * b + 1] < e0 ? h[2 * b + 1] : e0;
      mean += (double)(h[2 * b + 1] - h[2 * b]) / grid;
    }
    fprintf(stderr, "[gram ctatime] span %.3f ms, first CTA done at %.3f ms, mean CTA %.3f ms\n", (e1 - s0) * 1e-6,
            (e0 - s0) * 1e-6, mean * 1e-6);
  }
  if (rc == PF_OK && P.wlist) {  // the split 128 / 32-row items (a device-side list, maybe empty)
    TileParams W = P;
    W.kt_max = kGramKt;
    rc = run_tile_ws(W, st);
  }
  if (debug && rc == PF_OK) {
    static unsigned long long h[32 * 1024];
    cudaMemcpyAsync(h, dbg, sizeof(unsigned long long) * 32 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[24] = {"load:b_empty", "mma:r_empty(gram)", "mma:b_full(gram)", "mma:b_full(G)", "mma:a_full",
                             "mma:r_empty(blk)", "build:a_empty", "acc:r_full(gram)", "acc:r_full(blk)", "build:busy",
                             "acc:busy", "total", "build:item", "build:coef", "build:bar", "build:units",
                             "build:st_wait", "acc:drain", "acc:fss", "acc:sload", "acc:bar_xss", "acc:softmax",
                             "acc:rest", "build:loop"};
    fprintf(stderr, "[gram debug] mean cycles per CTA over %d CTAs:", grid);
    for (int q = 0; q < 24; ++q) {
      double sum = 0;
      for (int b = 0; b < grid; ++b) sum += (double)h[b * 32 + q];
      fprintf(stderr, " %s=%.3g", names[q], sum / grid);
    }
    double tmin = 1e300, tmax = 0;  // per-CTA spread of the total (static item striding)
    for (int b = 0; b < grid; ++b) {
      tmin = h[b * 32 + 11] < tmin ? (double)h[b * 32 + 11] : tmin;
      tmax = h[b * 32 + 11] > tmax ? (double)h[b * 32 + 11] : tmax;
    }
    fprintf(stderr, " total_min=%.3g total_max=%.3g\n", tmin, tmax);
  }
  return rc;
}

}  // namespace tile
}  // namespace pf

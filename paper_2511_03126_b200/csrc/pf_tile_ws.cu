// Persistent, warp-specialised tcgen05 tile kernel of the bf16 fused query (see pf_tile.cu for the
// formulation). One CTA per SM loops over tiles of 128 sorted points. Roles (24 warps, 6 warp
// groups; setmaxnreg moves registers from the producer groups to the accumulator groups):
//
//   warps 0-5   B loaders: for every 64-channel chunk of a tile (D/64 feature chunks, then the two
//               G-table chunks) they copy each tap's 128-byte row piece with cp.async (16 B per
//               lane op, 8 lanes per row; each thread keeps its rows' cell offsets in registers)
//               into a 6-stage ring of B buffers (N-major, 128-byte swizzle), three chunks in
//               flight; after cp.async.wait_group each warp fences the generic->async proxy and
//               arrives once on the stage's full barrier.
//   warp 6      MMA issuer: one elected thread copies the tile's A (bilinear weights) from shared
//               memory into TMEM (tcgen05.cp) and issues tcgen05.mma (M=128, N=128 = two chunks,
//               K=16, A from TMEM) into 3 rotating TMEM accumulator slots (feature chunk pairs and
//               the final similarity pair share the rotation); tcgen05.commit frees B stages and
//               signals the accumulators.
//   warp 7      idle (fills the warp group).
//   warps 8-15  accumulators (two per TMEM lane group, each half of the columns): |F|^2 from every
//               feature chunk pair (optional mean features), then one pass over the similarity
//               columns for softmax sums and property regression and a second for the weight
//               totals, which stay in registers across all tiles of the CTA; voxel atomics; the
//               regressed properties go to the sorted records.
//   warps 16-23 A builders (two threads per tile row, alternating over the row's visible views):
//               build the next tile's W (bilinear weights, bf16, K-major 128-B swizzle) while the
//               current tile's MMAs run.
// Synchronisation is mbarrier-only (full/empty pairs for A, B stages and TMEM accumulator slots).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "pf_common.cuh"
#include "pf_tc.cuh"
#include "pf_tile.cuh"
#include "pf_tile_dev.cuh"

namespace pf {
namespace tile {
namespace {

constexpr int kLoadWarps = 6;          // warps 0-5: B loaders
constexpr int kLoadThreads = 32 * kLoadWarps;
constexpr int kMmaWarp = 6;            // warp 6: MMA issuer (warp 7 idle)
constexpr int kAccWarp0 = 8;           // warps 8-15: accumulators (2 per TMEM lane group)
constexpr int kAccThreads = 256;
constexpr int kBuildWarp0 = 16;        // warps 16-23: A builders (two per tile row)
constexpr int kBuildWarps = 8;
constexpr int kBuildThreads = 32 * kBuildWarps;
constexpr int kWsThreads = 768;        // 24 warps = 6 warp groups
constexpr int kCG = 2;                 // 64-column B chunks per MMA group (N = 64 * kCG)
constexpr int kDCols = 64 * kCG;       // TMEM columns of one accumulator slot
constexpr int kDBufs = 3;              // TMEM accumulator slots (feature groups and the S group rotate)
constexpr int kStages = 6;             // B ring depth (3 chunk groups)
constexpr int kKtWs = 192;             // taps per tile held in one A buffer / B stage
constexpr int kStageBytes = kKtWs * 128;
constexpr int kABytes = kTile * ((kKtWs + 63) / 64) * 64 * 2;  // whole 64-column swizzle atoms
constexpr int kRowStep = kLoadThreads / 8;                      // rows between one thread's copies
constexpr int kRowsPer = kKtWs / kRowStep;                      // copies per thread per chunk
constexpr int kHalfK = kMaxKpadTC / 2;                          // materials per accumulator half
constexpr int kRegLaunch = 80;                                  // 65536 / 768, rounded down to 8
constexpr int kRegProducer = 48, kRegAcc = 136;                 // setmaxnreg budgets (6 x 128 threads)
static_assert(4 * 128 * kRegProducer + 2 * 128 * kRegAcc <= kWsThreads * kRegLaunch, "register pool");
static_assert(kRowStep % 8 == 0, "a thread's rows keep their swizzle phase");

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

struct WsShared {
  uint64_t a_full, a_empty;
  uint64_t b_full[kStages], b_empty[kStages];
  uint64_t d_full[kDBufs], d_empty[kDBufs];
  uint32_t tmem_base;
  int pad;
  uint2 desc_a[kMaxViewsTC];     // A builders' copy of the tile windows
  int32_t cell[2][kKtWs];        // loaders: tap row -> global cell, per tile (ring of 2)
  ViewF sv[kMaxViewsTC];
  float4 yv[kMaxKpadTC];         // per material: {y0, y1, mid_theta, bias (0 | -inf for padding)}
  float4 yv2[kMaxKpadTC];        // per material: {y2, y3, 0, 0} (P > 2)
  float xss[2][kTile];           // accumulator halves: partial |F|^2
  float xm[2][kTile];            //                     partial max (large 1/T only)
  float xsum[2][6][kTile];       //                     partial softmax sums
  double red[kMaxKpadTC + 8];
};

__device__ __forceinline__ int tile_ktp(const TileParams& P, int64_t tile, bool& ok) {
  const int kt = P.tile_kt[tile];
  const int ktp = (kt + 15) & ~15;
  ok = kt > 0 && ktp <= kKtWs;
  return ktp;
}

__device__ __forceinline__ uint16_t f2bf16(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool PROF>
__global__ void __launch_bounds__(kWsThreads, 1) k_tile_ws(const __grid_constant__ TileParams P, int need_max) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;                     // [128 rows x kKtWs] bf16
  unsigned char* sB = smem + kABytes;           // kStages x [kKtWs rows x 128 B]
  __shared__ WsShared S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nd = P.d >> 6, ns = P.kpadg >> 6, nch = nd + ns;
  const int64_t ntiles = (P.n + kTile - 1) / kTile;
  // PROF (PF_WS_DEBUG=1): per-role mbarrier wait / issue cycles, printed by the host
  long long wait_cyc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long issue_cyc = 0;
  const long long t_start = PROF ? clock64() : 0;
#define WS_WAIT(bar, par, slot)                    \
  do {                                             \
    if constexpr (PROF) {                          \
      const long long t0_ = clock64();             \
      tc::mbar_wait_or_trap(bar, par, slot);       \
      wait_cyc[slot] += clock64() - t0_;           \
    } else {                                       \
      tc::mbar_wait(bar, par);                     \
    }                                              \
  } while (0)
#define WS_CLOCK() (PROF ? clock64() : 0ll)

  // ---- setup ------------------------------------------------------------------------------------------
  for (int j = tid; j < P.nv; j += kWsThreads) S.sv[j] = make_viewf(P.views[j], P.d);
  for (int j = tid; j < kMaxKpadTC; j += kWsThreads) {
    float y[4];
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) y[pp] = (pp < P.p && j < P.k) ? P.values[j * P.p + pp] : 0.f;
    S.yv[j] = make_float4(y[0], y[1], j < P.k ? P.mid_theta[j] : 0.f, j < P.k ? 0.f : -INFINITY);
    S.yv2[j] = make_float4(y[2], y[3], 0.f, 0.f);
  }
  for (int j = tid; j < kMaxKpadTC + 8; j += kWsThreads) S.red[j] = 0.0;
  if (tid == 0) {
    tc::mbar_init(&S.a_full, kBuildWarps);
    tc::mbar_init(&S.a_empty, 1);
    for (int b = 0; b < kDBufs; ++b) {
      tc::mbar_init(&S.d_full[b], 1);
      tc::mbar_init(&S.d_empty[b], kAccThreads / 32);
    }
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.b_full[s], kLoadWarps);
      tc::mbar_init(&S.b_empty[s], 1);
    }
  }
  if (warp == kAccWarp0) tc::tmem_alloc(&S.tmem_base, 512);
  static_assert(kDBufs * kDCols + kKtWs / 2 <= 512, "TMEM: accumulator slots + A");
  static_assert(kDCols == kMaxKpadTC, "the S group fills one accumulator slot");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  const uint32_t tA = tbase + kDBufs * kDCols;          // A (bf16 pairs): kKtWs / 2 columns

  if (warp < kLoadWarps) {
    // ================= B loaders =================
    reg_dealloc<kRegProducer>();
    // thread -> 16-byte column q of rows r0, r0 + kRowStep, ...; pad rows repeat row 0's cell
    const int q = tid & 7, r0 = tid >> 3;
    int stage = 0;
    uint32_t phase = 0;
    int npend = 0;   // chunks whose cp.async groups are in flight: stages stage-npend .. stage-1
    uint32_t t_local = 0;
    auto retire_oldest = [&](int keep) {  // wait for the oldest group, publish its stage
      const long long tr0 = WS_CLOCK();
      if (keep == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (keep == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      if constexpr (PROF) wait_cyc[10] += clock64() - tr0;
      tc::fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.b_full[(stage + kStages - npend) % kStages]);
      --npend;
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      // row -> cell table for this tile
      int32_t* cell = S.cell[t_local & 1];
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      for (int v = tid; v < P.nv; v += kLoadThreads) {
        const uint2 ds = P.tile_desc[tile * P.nv + v];
        const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
        const int w = ds.y & 0xff, h = (ds.y >> 8) & 0xff;
        const ViewF& vw = S.sv[v];
        for (int a = 0; a < w * h; ++a) cell[base + a] = vw.cell_base + (y0 + a / w) * vw.Wf + x0 + a % w;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      const int kt = P.tile_kt[tile];
      int rc[kRowsPer];
#pragma unroll
      for (int j = 0; j < kRowsPer; ++j) {
        const int r = r0 + kRowStep * j;
        rc[j] = r < ktp ? cell[r < kt ? r : 0] : -1;
      }
      for (int c = 0; c < nch; ++c) {
        WS_WAIT(&S.b_empty[stage], phase ^ 1u, 0);
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
        // rows r0 + kRowStep*j: r & 7 is fixed per thread, so the swizzled destination advances by
        // kRowStep/8 row groups of 1024 bytes per copy
        const uint32_t dst0 = sb + (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + (((q ^ (r0 & 7)) & 7) << 4));
        const long long tl0 = WS_CLOCK();
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j)
          if (rc[j] >= 0) tc::cp_async16(dst0 + (uint32_t)j * (kRowStep / 8 * 1024u), src + (int64_t)rc[j] * rowlen);
        asm volatile("cp.async.commit_group;" ::: "memory");
        if constexpr (PROF) wait_cyc[11] += clock64() - tl0;
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
        if (++npend == 3) retire_oldest(2);
      }
      ++t_local;
    }
    while (npend > 0) retire_oldest(npend - 1);
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    // chunks are issued in pairs: two consecutive 64-column B chunks sit in adjacent ring stages
    // (the pair always starts on an even stage: D/64 and the 2 G chunks are even), so one MMA
    // covers N = 128 with LBO = stage stride.
    reg_dealloc<kRegProducer>();
    int stage = 0;
    uint32_t phase = 0;
    uint32_t dcount = 0;  // chunk pairs issued so far (selects the TMEM accumulator slot)
    uint32_t t_local = 0;
    const uint32_t idesc = tc::idesc_bf16_f32(128, kDCols, false, true);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      WS_WAIT(&S.a_full, t_local & 1u, 1);
      const uint32_t a0 = tc::smem_u32(sA);
      // A (the tile's bilinear weights) into TMEM once per tile (tcgen05.cp, 128 rows x 16 k per
      // op); the MMAs then read A from TMEM and only B from shared memory. The copies execute in
      // issue order after the previous tile's MMAs, so one TMEM A region suffices; the commit
      // releases the shared-memory A buffer to the builders as soon as the copies are done.
      tc::fence_after_sync();
      if (lane == 0) {
        for (int s = 0; s < ktp / 16; ++s)
          tc::tmem_cp_128x256b(tA + (uint32_t)(s * 8),
                               tc::smem_desc_sw128(a0 + (s >> 2) * kTile * 128 + (s & 3) * 32, 16, 1024));
        tc::mma_commit(&S.a_empty);
      }
      __syncwarp();
      for (int c = 0; c < nch; c += kCG) {
#pragma unroll
        for (int g = 0; g < kCG; ++g) WS_WAIT(&S.b_full[stage + g], phase, 2);
        const int db = dcount % kDBufs;
        if (c < nd) WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 3);
        else WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 4);
        const uint32_t dst = tbase + (uint32_t)(db * kDCols);
        tc::fence_after_sync();
        const long long ti0 = WS_CLOCK();
        if (lane == 0) {
          // (loaders and builders fence their generic-proxy writes before arriving)
          const uint32_t b0 = tc::smem_u32(sB + stage * kStageBytes);
          for (int s = 0; s < ktp / 16; ++s) {
            const uint64_t bd = tc::smem_desc_sw128(b0 + s * 2048, kStageBytes, 1024);
            tc::mma_bf16_ts(dst, tA + (uint32_t)(s * 8), bd, idesc, s > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int g = 0; g < kCG; ++g) tc::mma_commit(&S.b_empty[stage + g]);
          tc::mma_commit(&S.d_full[db]);
        }
        __syncwarp();
        if constexpr (PROF) issue_cyc += clock64() - ti0;
        ++dcount;
        stage += kCG;
        if (stage == kStages) { stage = 0; phase ^= 1u; }
      }
      ++t_local;
    }
  } else if (warp < kAccWarp0) {
    reg_dealloc<kRegProducer>();  // idle warp of the second group
  } else if (warp >= kBuildWarp0) {
    // ================= A builders (two threads per tile row) =================
    reg_dealloc<kRegProducer>();
    const int bt = tid - kBuildWarp0 * 32;   // 0..255
    const int row = bt & (kTile - 1), hb = bt >> 7;
    uint32_t t_local = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      WS_WAIT(&S.a_empty, (t_local & 1u) ^ 1u, 5);
      uint2* sdesc = S.desc_a;
      for (int v = bt; v < P.nv; v += kBuildThreads) sdesc[v] = P.tile_desc[tile * P.nv + v];
      uint4* a4 = reinterpret_cast<uint4*>(sA);
      for (int e = bt; e < ((ktp + 63) >> 6) * kTile * 8; e += kBuildThreads) a4[e] = make_uint4(0, 0, 0, 0);
      asm volatile("bar.sync 1, %0;" ::"n"(kBuildThreads) : "memory");  // zeros + windows visible
      const int64_t jpt = tile * kTile + row;
      if (jpt < P.n) {
        const float4 p = P.spts[jpt];
        const uint2 mw = *reinterpret_cast<const uint2*>(P.srec + jpt);
        int nth = 0;
#pragma unroll
        for (int w = 0; w < 2; ++w) {
          uint32_t bits = w ? mw.y : mw.x;
          while (bits) {
            const int v = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            if ((nth++ & 1) != hb) continue;  // the row's other thread takes this view
            const ProjF q = project_f32(S.sv[v], p.x, p.y, p.z);
            const TapF t = taps_f32(S.sv[v], q.u, q.v);
            float w00 = (1.f - t.wy) * (1.f - t.wx), w01 = (1.f - t.wy) * t.wx;
            float w10 = t.wy * (1.f - t.wx), w11 = t.wy * t.wx;
            if (!t.dx) { w00 += w01; w10 += w11; }
            if (!t.dy) { w00 += w10; w01 += w11; }
            const uint2 ds = sdesc[v];
            const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
            const int ww = ds.y & 0xff;
            const int c00 = base + (t.y0 - y0) * ww + (t.x0 - x0);
            *reinterpret_cast<uint16_t*>(sA + tc::a_off(row, c00, kTile)) = f2bf16(w00);
            if (t.dx) *reinterpret_cast<uint16_t*>(sA + tc::a_off(row, c00 + 1, kTile)) = f2bf16(w01);
            if (t.dy) *reinterpret_cast<uint16_t*>(sA + tc::a_off(row, c00 + ww, kTile)) = f2bf16(w10);
            if (t.dx && t.dy) *reinterpret_cast<uint16_t*>(sA + tc::a_off(row, c00 + ww + 1, kTile)) = f2bf16(w11);
          }
        }
      }
      tc::fence_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.a_full);
      ++t_local;
    }
  } else {
    // ================= accumulators: two warps per TMEM lane group, split by columns =================
    reg_alloc<kRegAcc>();
    const int half = (warp - kAccWarp0) >> 2;          // 0 / 1
    const int row = 32 * (warp & 3) + lane;            // TMEM lane = tile row
    const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int k0 = half * kHalfK;
    uint32_t dcount = 0;
    float wacc[kHalfK];  // weight totals of this thread's rows (integrate.py:133), all tiles
#pragma unroll
    for (int q = 0; q < kHalfK; ++q) wacc[q] = 0.f;
    double pm_sum = 0.0, pmx = 0.0, pmy = 0.0, pmz = 0.0, featured_n = 0.0, pairs = 0.0;
    const bool outs = P.sims || P.weights;
    const bool p_wide = P.p > 2;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      tile_ktp(P, tile, ok);
      const int64_t jpt = tile * kTile + row;
      const bool valid = jpt < P.n;
      if (!ok) {
        if (valid && half == 0) P.ovf_list[atomicAdd(P.ovf_count, 1)] = __float_as_int(P.spts[jpt].w);
        continue;
      }
      uint4 rec = make_uint4(0u, 0u, 0u, 0u);
      if (valid) rec = *reinterpret_cast<const uint4*>(P.srec + jpt);
      const int count = (int)rec.z;
      const float invc = count > 0 ? 1.f / (float)count : 0.f;
      const int32_t i = (valid && (outs || P.features)) ? __float_as_int(P.spts[jpt].w) : 0;
      float ss0 = 0.f, ss1 = 0.f, ss2 = 0.f, ss3 = 0.f;
      for (int c = 0; c < nd; c += kCG) {  // kCG chunks: this half drains kDCols / 2 columns
        const int db = dcount % kDBufs;
        WS_WAIT(&S.d_full[db], (dcount / kDBufs) & 1u, 6);
        tc::fence_after_sync();
#pragma unroll
        for (int g = 0; g < kCG; ++g) {  // 32 columns at a time (register budget: wacc stays live)
          float v[32];
          tc::tmem_ld32(tbase + (uint32_t)(db * kDCols + half * (kDCols / 2) + 32 * g) + t_lane, v);
          if (g == kCG - 1) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.d_empty[db]);  // data is in registers: release the slot
          }
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            ss0 = fmaf(v[q], v[q], ss0);
            ss1 = fmaf(v[q + 1], v[q + 1], ss1);
            ss2 = fmaf(v[q + 2], v[q + 2], ss2);
            ss3 = fmaf(v[q + 3], v[q + 3], ss3);
          }
          if (P.features && valid) {
            float* dst = P.features + (int64_t)i * P.d + c * 64 + half * (kDCols / 2) + 32 * g;
#pragma unroll
            for (int q = 0; q < 32; q += 4)
              *reinterpret_cast<float4*>(dst + q) =
                  make_float4(v[q] * invc, v[q + 1] * invc, v[q + 2] * invc, v[q + 3] * invc);
          }
        }
        ++dcount;
      }
      S.xss[half][row] = (ss0 + ss1) + (ss2 + ss3);
      // ---- epilogue on S (this half's materials) ----------------------------------------------------
      const int sslot = dcount % kDBufs;
      WS_WAIT(&S.d_full[sslot], (dcount / kDBufs) & 1u, 7);
      const uint32_t tS = tbase + (uint32_t)(sslot * kDCols + k0) + t_lane;
      tc::fence_after_sync();
      asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
      const float ss = S.xss[0][row] + S.xss[1][row];
      const bool featured = valid && count > 0;
      const float inv = ss > 0.f ? rsqrtf(ss) : 0.f;
      const float sc = inv * P.inv_temp * 1.4426950408889634f;  // log2(e) / (T |F|)
      // |s| <= 1 (cosines), so exp(s / T) cannot overflow for T >= ~0.013 and the row max of the
      // reference's stable softmax (grounding.py:175-177) only changes rounding; below that the
      // max is subtracted as in the reference (host sets need_max).
      float m2 = 0.f;
      if (need_max) {
        float mx = -INFINITY;
#pragma unroll
        for (int c0 = 0; c0 < kHalfK; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tS + (uint32_t)c0, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) mx = fmaxf(mx, fmaf(v[q], sc, S.yv[k0 + c0 + q].w));
        }
        S.xm[half][row] = mx;
        asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
        m2 = fmaxf(S.xm[0][row], S.xm[1][row]);
        if (!(m2 > -INFINITY)) m2 = 0.f;
      }
      float se = 0.f, pl0 = 0.f, pl1 = 0.f, pl2 = 0.f, pl3 = 0.f, pml = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < kHalfK; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tS + (uint32_t)c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const float4 y = S.yv[k0 + c0 + q];
          const float e = ex2(fmaf(v[q], sc, y.w - m2));  // padding columns: bias -inf -> 0
          se += e;
          pl0 = fmaf(e, y.x, pl0);
          pl1 = fmaf(e, y.y, pl1);
          pml = fmaf(e, y.z, pml);
        }
        if (p_wide) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float4 y = S.yv[k0 + c0 + q], y2 = S.yv2[k0 + c0 + q];
            const float e = ex2(fmaf(v[q], sc, y.w - m2));
            pl2 = fmaf(e, y2.x, pl2);
            pl3 = fmaf(e, y2.y, pl3);
          }
        }
      }
      S.xsum[half][0][row] = se;
      S.xsum[half][1][row] = pl0;
      S.xsum[half][2][row] = pl1;
      S.xsum[half][3][row] = pl2;
      S.xsum[half][4][row] = pl3;
      S.xsum[half][5][row] = pml;
      asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
      const float se_t = S.xsum[0][0][row] + S.xsum[1][0][row];
      if (featured && isnan(se_t)) atomicOr(P.status, 1);  // NaN similarity (grounding.py:173-174)
      const float rs = featured ? 1.f / se_t : 0.f;
      // normalised weights of this half -> per-thread weight totals (columns >= K are never read)
#pragma unroll
      for (int c0 = 0; c0 < kHalfK; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tS + (uint32_t)c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) wacc[c0 + q] = fmaf(ex2(fmaf(v[q], sc, -m2)), rs, wacc[c0 + q]);
      }
      if (outs) {  // validation outputs (similarities, softmax weights), caller's order
        for (int c0 = 0; c0 < kHalfK; c0 += 32) {
          float v[32];
          tc::tmem_ld32(tS + (uint32_t)c0, v);  // warp-collective: every lane, valid or not
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            if (!valid || k0 + c0 + q >= P.k) continue;
            if (P.sims) P.sims[(int64_t)i * P.k + k0 + c0 + q] = featured ? v[q] * inv : 0.f;
            if (P.weights) P.weights[(int64_t)i * P.k + k0 + c0 + q] = ex2(fmaf(v[q], sc, -m2)) * rs;
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.d_empty[sslot]);
      ++dcount;
      if (valid && half == 0) {
        float prop[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) prop[pp] = (S.xsum[0][1 + pp][row] + S.xsum[1][1 + pp][row]) * rs;
        const float pm = (S.xsum[0][5][row] + S.xsum[1][5][row]) * rs;
        const float4 p = P.spts[jpt];
        *(reinterpret_cast<float4*>(P.srec + jpt) + 1) = make_float4(prop[0], prop[1], prop[2], prop[3]);
        if (P.grid_partials) {
          const int32_t code = (int32_t)rec.w;
          float rho = prop[0];
#pragma unroll
          for (int pp = 1; pp < 4; ++pp) rho = P.density_col == pp ? prop[pp] : rho;
          atomicAdd(P.grid_partials + code, rho);
          atomicAdd(P.grid_partials + P.cells3 + code, 1.0f);
        }
        pm_sum += pm;
        pmx += (double)pm * p.x;
        pmy += (double)pm * p.y;
        pmz += (double)pm * p.z;
        featured_n += featured ? 1.0 : 0.0;
        pairs += count;
      }
    }
    // flush this CTA's partials (integrate.py:133-155) once
#pragma unroll
    for (int q = 0; q < kHalfK; ++q) {
      const float s = warp_sum(wacc[q]);
      if (lane == 0 && k0 + q < P.k && s != 0.f) atomicAdd(&S.red[k0 + q], (double)s);
    }
    double r6[6] = {pm_sum, pmx, pmy, pmz, featured_n, pairs};
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      r6[q] = warp_sum(r6[q]);
      if (lane == 0) atomicAdd(&S.red[P.k + q], r6[q]);
    }
    asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
    for (int j = tid - kAccWarp0 * 32; j < P.k + 6; j += kAccThreads)
      if (S.red[j] != 0.0) atomicAdd(P.partials + j, S.red[j]);
  }
  if (PROF && P.dbg && lane == 0 && (warp == 0 || warp == kMmaWarp || warp == kAccWarp0 || warp == kBuildWarp0)) {
    unsigned long long* d = P.dbg + blockIdx.x * 16;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (wait_cyc[q]) d[q] = (unsigned long long)wait_cyc[q];
    if (warp == 0) {
      d[10] = (unsigned long long)wait_cyc[10];
      d[11] = (unsigned long long)wait_cyc[11];
    }
    if (warp == kMmaWarp) {
      d[8] = (unsigned long long)(clock64() - t_start);
      d[9] = (unsigned long long)issue_cyc;
    }
  }
#undef WS_WAIT
#undef WS_CLOCK
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kAccWarp0) tc::tmem_dealloc(tbase, 512);
}

}  // namespace

int ws_kt_max() { return kKtWs; }

size_t ws_smem_bytes() { return (size_t)kABytes + (size_t)kStages * kStageBytes + 1024; }

// Launch the persistent kernel (one CTA per SM).
int run_tile_ws(const TileParams& P, cudaStream_t st) {
  if (P.kpadg != kMaxKpadTC) return set_error(PF_ERR_VALUE, "tile_ws: S operand must be %d wide", kMaxKpadTC);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = ws_smem_bytes();
  cudaFuncSetAttribute(k_tile_ws<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (P.n + kTile - 1) / kTile;
  int grid = (int)(ntiles < sms ? ntiles : sms);
  if (const char* g = getenv("PF_WS_GRID")) grid = (int)(ntiles < atoi(g) ? ntiles : atoi(g));  // debug knob
  // exp(s / T) with |s| <= 1 (+ bf16 rounding of G) stays below 2^120 unless T < ~0.012
  const int need_max = (double)P.inv_temp * 1.4426950408889634 * 1.05 > 120.0 ? 1 : 0;
  static unsigned long long* dbg = nullptr;
  TileParams Q = P;
  const bool debug = getenv("PF_WS_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 16 * 1024);
    cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 16 * 1024, st);
    Q.dbg = dbg;
  }
  if (debug) k_tile_ws<true><<<grid, kWsThreads, smem, st>>>(Q, need_max);
  else k_tile_ws<false><<<grid, kWsThreads, smem, st>>>(Q, need_max);
  const int rc = check_launch("tile_ws");
  if (debug && rc == PF_OK) {
    static unsigned long long h[16 * 1024];
    cudaMemcpyAsync(h, dbg, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[12] = {"load:b_empty", "mma:a_full", "mma:b_full", "mma:d_empty(F)", "mma:d_empty(S)",
                             "build:a_empty", "acc:d_full(F)", "acc:d_full(S)", "total", "mma:issue",
                             "load:retire", "load:issue"};
    fprintf(stderr, "[ws debug] mean cycles per CTA over %d CTAs:", grid);
    for (int q = 0; q < 12; ++q) {
      double sum = 0;
      for (int b = 0; b < grid; ++b) sum += (double)h[b * 16 + q];
      fprintf(stderr, " %s=%.3g", names[q], sum / grid);
    }
    fprintf(stderr, "\n");
  }
  return rc;
}

}  // namespace tile
}  // namespace pf

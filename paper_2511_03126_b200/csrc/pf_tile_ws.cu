// Persistent, warp-specialised tcgen05 tile kernel of the bf16 fused query (see pf_tile.cu for the
// formulation). One CTA per SM loops over tiles of 128 sorted points; roles (17 warps):
//
//   warps 0-3   B loaders: for every 64-channel chunk of a tile (D/64 feature chunks, then the
//               G-table chunks) they copy each tap's 128-byte row piece with cp.async (16 B per
//               lane op, 8 lanes per row) into a 4-stage ring of B buffers (N-major, 128-byte
//               swizzle), keeping three chunks in flight; after cp.async.wait_group the writer
//               fences the generic->async proxy and arrives on the stage's full barrier.
//               (Per-window TMA boxes were measured first: ~460 tiny TMA ops per tile made the TMA
//               unit the bottleneck, profiles/r01_notes.md.)
//   warp 4      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=64, K=16) over the
//               tile's taps into 4 TMEM buffers (feature chunks) or the S columns (G chunks);
//               tcgen05.commit frees the B stage / A buffer and signals the accumulators;
//   warps 5-12  accumulator warps (two per TMEM lane group, each half of the columns): drain each feature chunk from TMEM (|F|^2, optional mean
//               features), then the epilogue: softmax over K, property regression, voxel atomics,
//               integrate partials accumulated in registers across all tiles of the CTA;
//   warps 13-16 A builders: build the next tile's W (bilinear weights, bf16, K-major 128-B swizzle)
//               in one of two A buffers while the current tile's MMAs run.
// Synchronisation is mbarrier-only (full/empty pairs for A, B stages, TMEM D buffers and S).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "pf_common.cuh"
#include "pf_tc.cuh"
#include "pf_tile.cuh"
#include "pf_tile_dev.cuh"

namespace pf {
namespace tile {
namespace {

constexpr int kLoadWarps = 6;          // warps 0-5: B loaders
constexpr int kLoadThreads = 32 * kLoadWarps;
constexpr int kMmaWarp = 6;            // warp 6: MMA issuer
constexpr int kAccWarp0 = 7;           // warps 7-14: accumulators (2 per TMEM lane group)
constexpr int kAccThreads = 256;
constexpr int kBuildWarp0 = 15;        // warps 15-18: A builders
constexpr int kWsThreads = 608;        // 19 warps
constexpr int kCG = 2;                 // 64-column B chunks per MMA group (N = 64 * kCG)
constexpr int kDCols = 64 * kCG;       // TMEM columns of one feature buffer
constexpr int kDBufs = 3;              // TMEM accumulator slots (feature groups and the S group rotate)
constexpr int kStages = 6;             // B ring depth (3 chunk groups)
constexpr int kKtWs = 192;             // taps per tile held in one A buffer / B stage
constexpr int kStageBytes = kKtWs * 128;
constexpr int kABytes = kTile * ((kKtWs + 63) / 64) * 64 * 2;  // whole 64-column swizzle atoms
constexpr int kMaxBox = 4;             // TMA window boxes up to 4 x 4 cells

struct TMaps {
  CUtensorMap fm[kMaxBox * kMaxBox];
  CUtensorMap g[kMaxBox * kMaxBox];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(tc::smem_u32(bar))
      : "memory");
}

struct WsShared {
  uint64_t a_full[2], a_empty[2];
  uint64_t b_full[kStages], b_empty[kStages];
  uint64_t d_full[kDBufs], d_empty[kDBufs];
  uint64_t s_full, s_empty;
  uint32_t tmem_base;
  int pad;
  uint2 desc_a[2][kMaxViewsTC];  // A builders' copy of the tile windows, per A buffer
  int32_t cell[2][kKtWs];        // loaders: tap row -> global cell, per tile (ring of 2)
  ViewF sv[kMaxViewsTC];
  alignas(16) float svals[kMaxKpadTC * 4];  // read as float4
  float smt[kMaxKpadTC];
  float xss[2][kTile];           // accumulator halves: partial |F|^2
  float xm[2][kTile];            //                     partial max
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

__global__ void __launch_bounds__(kWsThreads, 1) k_tile_ws(const __grid_constant__ TileParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;                     // 2 x [128 rows x kKtWs] bf16
  unsigned char* sB = smem + kABytes;           // kStages x [kKtWs rows x 128 B]
  __shared__ WsShared S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nd = P.d >> 6, ns = P.kpadg >> 6, nch = nd + ns;
  const int64_t ntiles = (P.n + kTile - 1) / kTile;
  long long wait_cyc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long issue_cyc = 0;
  const long long t_start = clock64();
#define WS_WAIT(bar, par, slot)            \
  do {                                     \
    const long long t0_ = clock64();       \
    tc::mbar_wait(bar, par);               \
    wait_cyc[slot] += clock64() - t0_;     \
  } while (0)

  // ---- setup ------------------------------------------------------------------------------------------
  for (int j = tid; j < P.nv; j += kWsThreads) S.sv[j] = make_viewf(P.views[j], P.d);
  for (int j = tid; j < P.kpadg * 4; j += kWsThreads) {
    const int kk = j >> 2, pp = j & 3;
    S.svals[j] = (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f;
  }
  for (int j = tid; j < P.kpadg; j += kWsThreads) S.smt[j] = j < P.k ? P.mid_theta[j] : 0.f;
  for (int j = tid; j < kMaxKpadTC + 8; j += kWsThreads) S.red[j] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.a_full[b], 128);
      tc::mbar_init(&S.a_empty[b], 1);
    }
    for (int b = 0; b < kDBufs; ++b) {
      tc::mbar_init(&S.d_full[b], 1);
      tc::mbar_init(&S.d_empty[b], kAccThreads);
    }
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.b_full[s], kLoadThreads);
      tc::mbar_init(&S.b_empty[s], 1);
    }
    tc::mbar_init(&S.s_full, 1);
    tc::mbar_init(&S.s_empty, kAccThreads);
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
    // thread -> 16-byte column q of rows r0, r0 + 8, ...; pad rows repeat row 0's cell
    const int q = tid & 7, r0 = tid >> 3;
    int stage = 0;
    uint32_t phase = 0;
    int pending[3];  // stages whose cp.async groups are still in flight (oldest first)
    int npend = 0;
    uint32_t t_local = 0;
    auto retire_oldest = [&](int keep) {
      const long long tr0 = clock64();
      if (keep == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
      else if (keep == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      wait_cyc[10] += clock64() - tr0;
      tc::fence_async_shared();
      mbar_arrive(&S.b_full[pending[0]]);
      pending[0] = pending[1];
      pending[1] = pending[2];
      --npend;
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      // row -> cell table for this tile (ring of 2: the older slot's copies were all issued)
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
      for (int r = kt + tid; r < ktp; r += kLoadThreads) cell[r] = cell[0];
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      for (int c = 0; c < nch; ++c) {
        WS_WAIT(&S.b_empty[stage], phase ^ 1u, 0);
        const uint32_t sb = tc::smem_u32(sB + stage * kStageBytes);
        const uint16_t* src;
        int64_t rowlen;
        if (c < nd) {
          src = reinterpret_cast<const uint16_t*>(P.fmap) + c * 64 + q * 8;
          rowlen = P.d;
        } else {
          src = P.Gbf + (c - nd) * 64 + q * 8;
          rowlen = P.kpadg;
        }
        // rows r0, r0 + 8, ...: r & 7 is fixed per thread, so the swizzled destination just
        // advances by one 1024-byte row group per step (tc::b_chunk_off with the constant hoisted)
        static_assert(kLoadWarps % 2 == 0, "rows step by a multiple of 8");
        constexpr int kRowStep = kLoadThreads / 8;
        const uint32_t dst0 = sb + (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + (((q ^ (r0 & 7)) & 7) << 4));
        const int nrow = (ktp - r0 + kRowStep - 1) / kRowStep;
        const long long tl0 = clock64();
#pragma unroll 4
        for (int j = 0; j < nrow; ++j)
          tc::cp_async16(dst0 + (uint32_t)j * (kRowStep / 8 * 1024u), src + (int64_t)cell[r0 + kRowStep * j] * rowlen);
        asm volatile("cp.async.commit_group;" ::: "memory");
        wait_cyc[11] += clock64() - tl0;
        pending[npend++] = stage;
        if (npend == 3) retire_oldest(2);
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      }
      ++t_local;
    }
    while (npend > 0) retire_oldest(npend - 1);
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    // chunks are issued in pairs: two consecutive 64-column B chunks sit in adjacent ring stages
    // (the pair always starts on an even stage: D/64 and the 2 G chunks are even), so one MMA
    // covers N = 128 with LBO = stage stride — half the A re-reads of N = 64 MMAs.
    int stage = 0;
    uint32_t phase = 0;
    uint32_t dcount = 0;  // feature chunk pairs issued so far (selects the TMEM D buffer)
    uint32_t t_local = 0, s_phase = 0;
    const uint32_t idesc = tc::idesc_bf16_f32(128, kDCols, false, true);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      const int ab = 0;  // one shared-memory A buffer: it is free once the tcgen05.cp to TMEM is done
      WS_WAIT(&S.a_full[ab], t_local & 1u, 1);
      const uint32_t a0 = tc::smem_u32(sA + ab * kABytes);
      // A (the tile's bilinear weights) into TMEM once per tile (tcgen05.cp, 128 rows x 16 k per
      // op); the MMAs then read A from TMEM and only B from shared memory. The copies execute in
      // issue order after the previous tile's MMAs, so one TMEM A region suffices; the commit
      // releases the shared-memory A buffer to the builders as soon as the copies are done.
      tc::fence_after_sync();
      if (lane == 0) {
        for (int s = 0; s < ktp / 16; ++s)
          tc::tmem_cp_128x256b(tA + (uint32_t)(s * 8),
                               tc::smem_desc_sw128(a0 + (s >> 2) * kTile * 128 + (s & 3) * 32, 16, 1024));
        tc::mma_commit(&S.a_empty[ab]);
      }
      __syncwarp();
      for (int c = 0; c < nch; c += kCG) {
#pragma unroll
        for (int g = 0; g < kCG; ++g) WS_WAIT(&S.b_full[stage + g], phase, 2);
        uint32_t dst;
        int db = 0;
        db = dcount % kDBufs;  // feature groups and the final S group share the slot rotation
        if (c < nd) WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 3);
        else WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 4);
        dst = tbase + (uint32_t)(db * kDCols);
        tc::fence_after_sync();
        const long long ti0 = clock64();
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
        issue_cyc += clock64() - ti0;
        ++dcount;
        stage += kCG;
        if (stage == kStages) { stage = 0; phase ^= 1u; }
      }
      s_phase ^= 1u;
      ++t_local;
    }
  } else if (warp >= kBuildWarp0) {
    // ================= A builders (thread = tile row) =================
    const int row = tid - kBuildWarp0 * 32;  // 0..127
    uint32_t t_local = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      const int ktp = tile_ktp(P, tile, ok);
      if (!ok) continue;
      const int ab = 0;
      WS_WAIT(&S.a_empty[ab], (t_local & 1u) ^ 1u, 5);
      uint2* sdesc = S.desc_a[ab];
      for (int v = row; v < P.nv; v += 128) sdesc[v] = P.tile_desc[tile * P.nv + v];
      unsigned char* A = sA + ab * kABytes;
      uint4* a4 = reinterpret_cast<uint4*>(A);
      for (int e = row; e < ((ktp + 63) >> 6) * kTile * 8; e += 128) a4[e] = make_uint4(0, 0, 0, 0);
      asm volatile("bar.sync 1, 128;" ::: "memory");  // builders only: zeros + windows visible
      const int64_t jpt = tile * kTile + row;
      if (jpt < P.n) {
        const int32_t i = P.perm[jpt];
        const float4 p = P.spts[jpt];
        for (int w = 0; w < P.nwords; ++w) {
          uint32_t bits = P.mask_bits[(int64_t)i * P.nwords + w];
          while (bits) {
            const int v = w * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
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
            *reinterpret_cast<uint16_t*>(A + tc::a_off(row, c00, kTile)) = f2bf16(w00);
            if (t.dx) *reinterpret_cast<uint16_t*>(A + tc::a_off(row, c00 + 1, kTile)) = f2bf16(w01);
            if (t.dy) *reinterpret_cast<uint16_t*>(A + tc::a_off(row, c00 + ww, kTile)) = f2bf16(w10);
            if (t.dx && t.dy) *reinterpret_cast<uint16_t*>(A + tc::a_off(row, c00 + ww + 1, kTile)) = f2bf16(w11);
          }
        }
      }
      tc::fence_async_shared();
      mbar_arrive(&S.a_full[ab]);
      ++t_local;
    }
  } else {
    // ================= accumulator warps: two per TMEM lane group, split by columns =================
    const int half = (warp - kAccWarp0) >> 2;          // 0 / 1
    const int row = 32 * (warp & 3) + lane;            // TMEM lane = tile row
    const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int kh = P.kpadg >> 1;                       // materials per half (32 or 64)
    const int k0 = half * kh;
    uint32_t dcount = 0, s_phase = 0;
    float wt[2] = {0.f, 0.f};
    double pm_sum = 0.0, pmx = 0.0, pmy = 0.0, pmz = 0.0, featured_n = 0.0, pairs = 0.0;
    const float4* sv4 = reinterpret_cast<const float4*>(S.svals);
    const bool outs = P.sims || P.weights;
    const int p_n = P.p;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      bool ok;
      tile_ktp(P, tile, ok);
      const int64_t jpt = tile * kTile + row;
      const bool valid = jpt < P.n;
      const int32_t i = valid ? P.perm[jpt] : 0;
      if (!ok) {
        if (valid && half == 0) P.ovf_list[atomicAdd(P.ovf_count, 1)] = i;
        continue;
      }
      const int count = valid ? P.counts[i] : 0;
      const float invc = count > 0 ? 1.f / (float)count : 0.f;
      float ss0 = 0.f, ss1 = 0.f, ss2 = 0.f, ss3 = 0.f;
      for (int c = 0; c < nd; c += kCG) {  // kCG chunks: this half drains kDCols / 2 columns
        const int db = dcount % kDBufs;
        WS_WAIT(&S.d_full[db], (dcount / kDBufs) & 1u, 6);
        tc::fence_after_sync();
        float v[kCG][32];
#pragma unroll
        for (int g = 0; g < kCG; ++g)
          tc::tmem_ld32(tbase + (uint32_t)(db * kDCols + half * (kDCols / 2) + 32 * g) + t_lane, v[g]);
        tc::fence_before_sync();
        mbar_arrive(&S.d_empty[db]);  // data is in registers: release the buffer early
#pragma unroll
        for (int g = 0; g < kCG; ++g) {
#pragma unroll
          for (int q = 0; q < 32; q += 4) {
            ss0 = fmaf(v[g][q], v[g][q], ss0);
            ss1 = fmaf(v[g][q + 1], v[g][q + 1], ss1);
            ss2 = fmaf(v[g][q + 2], v[g][q + 2], ss2);
            ss3 = fmaf(v[g][q + 3], v[g][q + 3], ss3);
          }
          if (P.features && valid) {
            float* dst = P.features + (int64_t)i * P.d + c * 64 + half * (kDCols / 2) + 32 * g;
#pragma unroll
            for (int q = 0; q < 32; q += 4)
              *reinterpret_cast<float4*>(dst + q) =
                  make_float4(v[g][q] * invc, v[g][q + 1] * invc, v[g][q + 2] * invc, v[g][q + 3] * invc);
          }
        }
        ++dcount;
      }
      S.xss[half][row] = (ss0 + ss1) + (ss2 + ss3);
      // ---- epilogue on S (this half's materials) ----------------------------------------------------
      const int sslot = dcount % kDBufs;
      WS_WAIT(&S.d_full[sslot], (dcount / kDBufs) & 1u, 7);
      const uint32_t tS = tbase + (uint32_t)(sslot * kDCols);
      tc::fence_after_sync();
      float mx = -INFINITY;
      bool nan = false;
      for (int c0 = 0; c0 < kh; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tS + (uint32_t)(k0 + c0) + t_lane, v);
        if (k0 + c0 + 32 <= P.k) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            mx = fmaxf(mx, v[q]);
            nan |= isnan(v[q]);
          }
        } else {
          for (int q = 0; k0 + c0 + q < P.k; ++q) {
            mx = fmaxf(mx, v[q]);
            nan |= isnan(v[q]);
          }
        }
      }
      S.xm[half][row] = mx;
      asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
      const float ss = S.xss[0][row] + S.xss[1][row];
      const bool featured = valid && count > 0;
      const float inv = ss > 0.f ? 1.f / sqrtf(ss) : 0.f;
      const float sc = inv * P.inv_temp * 1.4426950408889634f;  // > 0 (or 0 when featureless)
      const float m2 = fmaxf(S.xm[0][row], S.xm[1][row]) * sc;
      if (featured && (nan || isnan(sc))) atomicOr(P.status, 1);
      float se = 0.f, pl0 = 0.f, pl1 = 0.f, pl2 = 0.f, pl3 = 0.f, pml = 0.f;
      for (int c0 = 0; c0 < kh; c0 += 32) {
        float v[32];
        tc::tmem_ld32(tS + (uint32_t)(k0 + c0) + t_lane, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int kk = k0 + c0 + q;
          const float e = kk < P.k ? ex2(fmaf(v[q], sc, -m2)) : 0.f;
          se += e;
          const float4 y = sv4[kk];
          pl0 = fmaf(e, y.x, pl0);
          pl1 = fmaf(e, y.y, pl1);
          if (p_n > 2) {
            pl2 = fmaf(e, y.z, pl2);
            pl3 = fmaf(e, y.w, pl3);
          }
          pml = fmaf(e, S.smt[kk], pml);
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
      const float rs = featured ? 1.f / se_t : 0.f;
      // normalised weights of this half -> column sums across the warp (butterfly) -> wt registers
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (g * 32 < kh) {
          float v[32];
          tc::tmem_ld32(tS + (uint32_t)(k0 + g * 32) + t_lane, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int kk = k0 + g * 32 + q;
            const float wv = (kk < P.k && featured) ? ex2(fmaf(v[q], sc, -m2)) * rs : 0.f;
            if (outs && valid && kk < P.k) {
              if (P.sims) P.sims[(int64_t)i * P.k + kk] = featured ? v[q] * inv : 0.f;
              if (P.weights) P.weights[(int64_t)i * P.k + kk] = wv;
            }
            v[q] = wv;
          }
          // reduce-scatter: after 5 steps lane l holds the warp's sum of column k0 + g*32 + l
#pragma unroll
          for (int hb = 16; hb >= 1; hb >>= 1) {
            const bool upper = (lane & hb) != 0;
#pragma unroll
            for (int q = 0; q < hb; ++q) {
              const float send = upper ? v[q] : v[q + hb];
              const float keep = upper ? v[q + hb] : v[q];
              v[q] = keep + __shfl_xor_sync(0xffffffffu, send, hb);
            }
          }
          wt[g] += v[0];
        }
      }
      tc::fence_before_sync();
      mbar_arrive(&S.d_empty[sslot]);
      ++dcount;
      if (valid && half == 0) {
        float prop[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) prop[pp] = (S.xsum[0][1 + pp][row] + S.xsum[1][1 + pp][row]) * rs;
        const float pm = (S.xsum[0][5][row] + S.xsum[1][5][row]) * rs;
        const float4 p = P.spts[jpt];
        for (int pp = 0; pp < p_n; ++pp) P.props[(int64_t)i * p_n + pp] = prop[pp];
        if (P.grid_partials) {
          const int32_t code = P.codes[i];
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
    for (int g = 0; g < 2; ++g)
      if (g * 32 < kh && k0 + g * 32 + lane < P.k) atomicAdd(&S.red[k0 + g * 32 + lane], (double)wt[g]);
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
  if (P.dbg && lane == 0 && (warp == 0 || warp == kMmaWarp || warp == kAccWarp0 || warp == kBuildWarp0)) {
    unsigned long long* d = P.dbg + blockIdx.x * 16;
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
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kAccWarp0) tc::tmem_dealloc(tbase, 512);
}

// ---- host: tensor maps --------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

bool encode_window_map(CUtensorMap* m, const void* base, int cols, int wf, int rows_total, int bw, int bh) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)wf, (cuuint64_t)rows_total};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)cols * 2 * wf};
  const cuuint32_t box[3] = {64u, (cuuint32_t)bw, (cuuint32_t)bh};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int ws_kt_max() { return kKtWs; }

size_t ws_smem_bytes() { return (size_t)kABytes + (size_t)kStages * kStageBytes + 1024; }

// Launch the persistent kernel (one CTA per SM).
int run_tile_ws(const TileParams& P, int hf, int wf, int nv, cudaStream_t st) {
  (void)hf;
  (void)wf;
  (void)nv;
  if (P.kpadg % 64 != 0) return -1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = ws_smem_bytes();
  cudaFuncSetAttribute(k_tile_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t ntiles = (P.n + kTile - 1) / kTile;
  int grid = (int)(ntiles < sms ? ntiles : sms);
  if (const char* g = getenv("PF_WS_GRID")) grid = (int)(ntiles < atoi(g) ? ntiles : atoi(g));  // debug knob
  static unsigned long long* dbg = nullptr;
  TileParams Q = P;
  const bool debug = getenv("PF_WS_DEBUG") != nullptr;
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, sizeof(unsigned long long) * 16 * 1024);
    cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 16 * 1024, st);
    Q.dbg = dbg;
  }
  k_tile_ws<<<grid, kWsThreads, smem, st>>>(Q);
  const int rc = check_launch("tile_ws");
  if (debug && rc == PF_OK) {
    static unsigned long long h[16 * 1024];
    cudaMemcpyAsync(h, dbg, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[12] = {"load:b_empty", "mma:a_full", "mma:b_full", "mma:d_empty", "mma:s_empty",
                             "build:a_empty", "acc:d_full", "acc:s_full", "total", "mma:issue",
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

// ---- diagnostic: TMA window load at an arbitrary 128-byte row offset ---------------------------------
namespace pf {
namespace tile {
namespace {
__global__ void k_tma_selftest(const __grid_constant__ CUtensorMap map, int x0, int y0, int row_off,
                               int rows, uint16_t* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (uint32_t)rows * 128u);
    tma_load_3d(tc::smem_u32(smem) + row_off * 128, &map, 0, x0, y0, &bar);
  }
  __syncthreads();
  tc::mbar_wait(&bar, 0);
  // un-swizzle by the absolute-address rule (chunk c of row r stored at chunk c ^ (r & 7))
  for (int e = threadIdx.x; e < rows * 64; e += blockDim.x) {
    const int r = row_off + e / 64, n = e % 64;
    const uint32_t off = r * 128 + ((((n >> 3) ^ (r & 7)) & 7) << 4) + (n & 7) * 2;
    out[e] = *reinterpret_cast<const uint16_t*>(smem + off);
  }
}
}  // namespace
}  // namespace tile
}  // namespace pf

extern "C" int pf_selftest_tma(const void* src_bf16, int32_t hf, int32_t wf, int32_t x0, int32_t y0,
                               int32_t bw, int32_t bh, int32_t row_off, void* out, void* stream) {
  using namespace pf::tile;
  CUtensorMap m;
  if (!encode_window_map(&m, src_bf16, 64, wf, hf, bw, bh))
    return pf::set_error(PF_ERR_CUDA, "selftest_tma: tensor map encode failed");
  k_tma_selftest<<<1, 128, 8 * 1024 + 1024, reinterpret_cast<cudaStream_t>(stream)>>>(
      m, x0, y0, row_off, bw * bh, reinterpret_cast<uint16_t*>(out));
  return pf::check_launch("selftest_tma");
}

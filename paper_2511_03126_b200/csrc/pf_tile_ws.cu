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
//   warps 16-23 A builders: write the next tile's W (bilinear weights, bf16 pairs) straight into
//               one of two TMEM A buffers with tcgen05.st (warp 16 + j: lane quarter j & 3, views of
//               rank parity j >> 2) while the current tile's MMAs run.
// Synchronisation is mbarrier-only (full/empty pairs for A, B stages and TMEM accumulator slots).
#include <type_traits>
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
constexpr int kBuildWarp0 = 16;        // warps 16-23: A builders (two per 32 tile rows)
constexpr int kBuildWarps = 8;
constexpr int kBuildThreads = 32 * kBuildWarps;
constexpr int kWsThreads = 768;        // 24 warps = 6 warp groups
constexpr float kAffineR = 12e-3f;     // tiles wider than 2 * kAffineR (m) build with the exact projection:
                                       // the expansion error is ~fx X / Z^3 r^2 <= ~0.05 px (0.4% of a C5 cell)
constexpr int kTraceCtas = 4, kTraceTiles = 64, kTraceEvents = 64;
constexpr int kCG = 2;                 // 64-column B chunks per MMA group (N = 64 * kCG)
constexpr int kDCols = 64 * kCG;       // TMEM columns of one accumulator slot
constexpr int kDBufs = kCG == 1 ? 5 : 2;  // TMEM accumulator slots (with the two A buffers: 512 columns)
constexpr int kSGroups = kMaxKpadTC / kDCols;  // similarity groups per tile (1 or 2)
constexpr int kStages = 8;             // B ring depth (4 chunk groups)
constexpr int kKtWs = 192;             // taps per tile held in one A buffer / B stage
constexpr int kStageBytes = kKtWs * 128;
// x3 (f32 maps): A hi and lo parts per buffer, kKtX3 taps each: 2 x 2 x kKtX3/2 TMEM columns; the
// B ring holds hi and lo stages of every chunk pair (4 stages per MMA group)
constexpr int kKtX3 = 128;
static_assert(kDBufs * kDCols + 2 * kKtX3 <= 512, "TMEM: accumulator slots + 2 x (hi, lo) A buffers");
static_assert(kStages % 4 == 0, "x3 groups of 4 stages never wrap the ring");
constexpr int kRowStep = kLoadThreads / 8;                      // rows between one thread's copies
constexpr int kRowsPer = kKtWs / kRowStep;                      // copies per thread per chunk
constexpr int kHalfK = kMaxKpadTC / 2;                          // materials per accumulator half
constexpr int kRegLaunch = 80;                                  // 65536 / 768, rounded down to 8
constexpr int kRegProducer = 48, kRegAcc = 144;                 // setmaxnreg budgets (6 x 128 threads)
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
  uint64_t a_full[2], a_empty[2];
  uint64_t b_full[kStages], b_empty[kStages];
  uint64_t d_full[kDBufs], d_empty[kDBufs];
  uint32_t tmem_base;
  int pad;
  uint2 desc_a[2][kMaxViewsTC];  // A builders' copy of the tile windows (per A buffer)
  int32_t cell[2][kKtWs];        // loaders: tap row -> global cell, per tile (ring of 2)
  ViewF sv[kMaxViewsTC];
  float4 vpk[kMaxViewsTC][5];    // builders: packed camera {R0 R1 R2 t0}{R3 R4 R5 t1}{R6 R7 R8 t2}{fx cx fy cy}{ru rv Wf-1 Hf-1}
  float4 vcoef[2][kMaxViewsTC][2];  // builders: fu, fv = c0 + g . (p - o) per view rank (per A buffer)
  int32_t vrank[2][kMaxViewsTC];    // builders: view | window base << 8, per rank
  int4 vwin[2][kMaxViewsTC];        // builders: window x0, y0, w, h per rank
  float bbox[2][4][6];              // builders: per lane group box of the tile's points
  float4 yp[kMaxKpadTC];         // per material pair (k, k+1), at k/2: {y0 y0' y1 y1'} then {mt mt' b b'}
  float2 yv2[kMaxKpadTC];        // per material: {y2, y3} (P > 2)
  float xss[2][kTile];           // accumulator halves: partial |F|^2
  float xm[2][kTile];            //                     partial max (large 1/T only)
  float xsum[2][6][kTile];       //                     partial softmax sums
  double red[kMaxKpadTC + 8];
};


// every role reads the next tile's inputs (tap count, windows, points, records) one tile ahead, so
// their DRAM latency overlaps the current tile
__device__ __forceinline__ int ktp_of(int kt, bool& ok, int kt_max) {
  const int ktp = (kt + 15) & ~15;
  ok = kt > 0 && ktp <= kt_max;
  return ktp;
}
// LIST: the Gram path's list of split items (P.wlist) instead of this kernel's own tiles / sub-tiles
// (a template parameter: the own-items instantiation carries none of the list logic)
template <bool LIST>
__device__ __forceinline__ int kt_at(const TileParams& P, int64_t tile, int64_t ntiles) {
  if constexpr (LIST) return tile < ntiles ? (P.wlist[tile].z >> 16) : 0;  // ntiles = list length here
  return tile < ntiles ? P.tile_kt[tile] : 0;
}
// descriptor row of work item t (the Gram path's list names the item whose windows it uses)
template <bool LIST>
__device__ __forceinline__ int64_t desc_item(const TileParams& P, int64_t t) {
  if constexpr (LIST) return P.wlist[t].x;
  return t;
}

// work item t -> (tile, first row, row count): tiles first, then the sub-tiles of overflow tiles
// (list mode: the entry's first row and row count, inside one 128-row tile)
template <bool LIST>
__device__ __forceinline__ int64_t item_tile(const TileParams& P, int64_t t, int64_t ntiles, int& rlo, int& rhi) {
  if constexpr (LIST) {
    const int4 e = P.wlist[t];
    rlo = e.y % kTile;
    rhi = rlo + (e.z & 0xffff);
    return e.y / kTile;
  }
  if (t < ntiles) {
    rlo = 0;
    rhi = kTile;
    return t;
  }
  const int64_t b = (t - ntiles) >> 2;
  rlo = kSubRows * (int)((t - ntiles) & 3);
  rhi = rlo + kSubRows;
  return P.sub_tiles[b];
}
// does work item t cover tile row `row` (and is the point real)?
template <bool LIST>
__device__ __forceinline__ bool item_row(const TileParams& P, int64_t t, int64_t ntiles, int row, int64_t& jpt) {
  int rlo, rhi;
  const int64_t tl = item_tile<LIST>(P, t, ntiles, rlo, rhi);
  jpt = tl * kTile + row;
  return row >= rlo && row < rhi && jpt < P.n;
}

__device__ __forceinline__ uint16_t f2bf16(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// prefetch loads that must issue where they are written (a plain load may be sunk by the compiler
// to its first use a whole tile later, putting its DRAM latency on the critical path)
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

// packed fp32 pairs (sm_100 FFMA2 / FADD2): half the FP32 instructions of the epilogue math
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

// warp reduce-scatter of 32 values per lane: afterwards lane l holds the sum over the warp's lanes of
// value l (recursive halving: at distance o a lane keeps the half of its range selected by lane & o)
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

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// PROF: wait accounting + trace (PF_WS_DEBUG); OUTS: validation outputs (features, similarities,
// softmax weights) -- a separate instantiation keeps their fully unrolled stores out of the hot code
template <bool PROF, bool OUTS, bool X3, bool LIST = false>
__global__ void __launch_bounds__(kWsThreads, 1) k_tile_ws(const __grid_constant__ TileParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sB = smem;                     // kStages x [kKtWs rows x 128 B]
  __shared__ WsShared S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nd = P.d >> 6, ns = P.kpadg >> 6, nch = nd + ns;
  const int64_t ntiles = (P.n + kTile - 1) / kTile;
  const int64_t nitems = LIST ? (int64_t)*P.wcount : ntiles + 4 * (int64_t)min(*P.sub_count, P.max_sub_tiles);
  // PROF (PF_WS_DEBUG=1): per-role mbarrier wait / issue cycles, printed by the host
  long long wait_cyc[15] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long issue_cyc = 0;
  const long long t_start = PROF ? clock64() : 0;
  // PROF trace: per-tile role timestamps (cycles since kernel start) of the first kTraceTiles tiles of
  // the first kTraceCtas CTAs (profiles/ws_trace.py); events: 0 build start, 1 build coefficients
  // ready, 2 build done, 3 mma A ready, 4 + g mma group g committed (g < 10), 14 loader tile start,
  // 15 + g loader group g issued, 25 + g acc group g ready (lane quarter 0 of the owning parity; the
  // last group is the similarity group), 35 + g acc F group g released, 45 after the |F|^2 exchange,
  // 46 pass 1 done, 47 after the sums exchange, 48 pass 2 done, 49 epilogue done (slot released)
  uint32_t* trace =
      (PROF && P.trace && blockIdx.x < kTraceCtas) ? P.trace + blockIdx.x * kTraceTiles * kTraceEvents : nullptr;
#define WS_TRACE(tl, ev)                                                                   \
  do {                                                                                     \
    if (PROF && trace && (tl) < (uint32_t)kTraceTiles && (ev) < kTraceEvents)              \
      trace[(tl) * kTraceEvents + (ev)] = (uint32_t)(clock64() - t_start);                 \
  } while (0)
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
  for (int j = tid; j < P.nv; j += kWsThreads) {
    const ViewF w = make_viewf(P.views[j], P.d);
    S.sv[j] = w;
    S.vpk[j][0] = make_float4(w.R[0], w.R[1], w.R[2], w.t[0]);
    S.vpk[j][1] = make_float4(w.R[3], w.R[4], w.R[5], w.t[1]);
    S.vpk[j][2] = make_float4(w.R[6], w.R[7], w.R[8], w.t[2]);
    S.vpk[j][3] = make_float4(w.fx, w.cx, w.fy, w.cy);
    S.vpk[j][4] = make_float4(w.ru, w.rv, (float)(w.Wf - 1), (float)(w.Hf - 1));
  }
  for (int j = tid; j < kMaxKpadTC; j += kWsThreads) {
    float y[4];
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) y[pp] = (pp < P.p && j < P.k) ? P.values[j * P.p + pp] : 0.f;
    S.yv2[j] = make_float2(y[2], y[3]);
  }
  // softmax shift. The reference subtracts each row's max (grounding.py:175-177); |s_k| <= |t_k| bounds
  // every exponent s_k / T by c = max_k |t_k| / T (in log2 units here), so subtracting the constant c
  // instead keeps the exponents in [-2c, 0]: no overflow, and the row's largest term cannot underflow
  // while 2c <= 120. Beyond that (tiny T or long text rows) the row max is subtracted per point.
  // The 1.05 margin covers the bf16 rounding of the text / G operands.
  float shift;
  {
    const float cbound = 1.05f * __ldg(P.tbound) * P.inv_temp * 1.4426950408889634f;
    shift = (2.f * cbound <= 120.f) ? -cbound : 0.f;  // NaN / inf bound: per-row max (acc branch)
  }
  for (int j = tid; j < kMaxKpadTC / 2; j += kWsThreads) {
    auto val = [&](int kk, int pp) { return (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f; };
    const int a = 2 * j, b = 2 * j + 1;
    S.yp[2 * j] = make_float4(val(a, 0), val(b, 0), val(a, 1), val(b, 1));
    S.yp[2 * j + 1] = make_float4(a < P.k ? P.mid_theta[a] : 0.f, b < P.k ? P.mid_theta[b] : 0.f,
                                  a < P.k ? shift : -INFINITY, b < P.k ? shift : -INFINITY);
  }
  for (int j = tid; j < kMaxKpadTC + 8; j += kWsThreads) S.red[j] = 0.0;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.a_full[b], kBuildWarps);
      tc::mbar_init(&S.a_empty[b], 1);
    }
    for (int b = 0; b < kDBufs; ++b) {
      tc::mbar_init(&S.d_full[b], 1);
      tc::mbar_init(&S.d_empty[b], kAccThreads / 64);  // the 4 warps of the owning parity
    }
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.b_full[s], kLoadThreads);  // one cp.async.mbarrier.arrive.noinc per loader thread
      tc::mbar_init(&S.b_empty[s], 1);
    }
  }
  if (warp == kAccWarp0) tc::tmem_alloc(&S.tmem_base, 512);
  static_assert(kDBufs * kDCols + 2 * (kKtWs / 2) <= 512, "TMEM: accumulator slots + 2 A buffers");
  static_assert(kSGroups * kDCols == kMaxKpadTC && (kSGroups == 1 || kSGroups == 2), "similarity groups");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = S.tmem_base;
  // two A buffers (bf16 pairs, lane = tile row, k ascending): kKtWs / 2 columns each
  const uint32_t tA0 = tbase + kDBufs * kDCols;

  if (warp < kLoadWarps) {
    // ================= B loaders =================
    reg_dealloc<kRegProducer>();
    // thread -> 16-byte column q of rows r0, r0 + kRowStep, ...; pad rows repeat row 0's cell
    const int q = tid & 7, r0 = tid >> 3;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t published = 0, pub_tile = 0, pub_group = 0;  // PROF trace bookkeeping (warp 0)
    uint32_t t_local = 0;
    int kt_nx = kt_at<LIST>(P, blockIdx.x, nitems);
    uint2 ds_nx = (tid < P.nv && blockIdx.x < nitems) ? P.tile_desc[desc_item<LIST>(P, blockIdx.x) * P.nv + tid]
                                                      : make_uint2(0u, 0u);
    for (int64_t tile = blockIdx.x; tile < nitems; tile += gridDim.x) {
      const int kt = kt_nx;
      const uint2 ds_cur = ds_nx;
      kt_nx = kt_at<LIST>(P, tile + gridDim.x, nitems);
      if (tid < P.nv && tile + gridDim.x < nitems) ds_nx = P.tile_desc[desc_item<LIST>(P, tile + gridDim.x) * P.nv + tid];
      bool ok;
      const int ktp = ktp_of(kt, ok, X3 ? kKtX3 : kKtWs);
      if (!ok) continue;
      // row -> cell table for this tile
      int32_t* cell = S.cell[t_local & 1];
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      static_assert(kMaxViewsTC <= kLoadThreads, "one window per loader thread");
      for (int v = tid; v < P.nv; v += kLoadThreads) {
        const uint2 ds = ds_cur;
        const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
        const int w = ds.y & 0xff, h = (ds.y >> 8) & 0xff;
        const ViewF& vw = S.sv[v];
        const int sz = (w * h + 1) & ~1;  // padding column (zero weights) reads a valid row
        PF_DCHECK(sz == 0 || (base + sz <= ktp && x0 + w <= vw.Wf && y0 + h <= vw.Hf), "window inside the item / map");
        for (int a = 0; a < sz; ++a) {
          const int aa = a < w * h ? a : 0;
          cell[base + a] = vw.cell_base + (y0 + aa / w) * vw.Wf + x0 + aa % w;
        }
      }
      asm volatile("bar.sync 3, %0;" ::"n"(kLoadThreads) : "memory");
      if (tid == 0) WS_TRACE(t_local, 14);
      int rc[kRowsPer];
#pragma unroll
      for (int j = 0; j < kRowsPer; ++j) {
        const int r = r0 + kRowStep * j;
        rc[j] = r < ktp ? cell[r < kt ? r : 0] : -1;
        PF_DCHECK(rc[j] < 0 || rc[j] < S.sv[P.nv - 1].cell_base + S.sv[P.nv - 1].Hf * S.sv[P.nv - 1].Wf, "tap row inside the maps");
      }
      const int nstage = X3 ? 2 * nch : nch;  // x3: per chunk pair [hi c][hi c+1][lo c][lo c+1]
      for (int qs = 0; qs < nstage; ++qs) {
        const int c = X3 ? 2 * (qs >> 2) + (qs & 1) : qs;
        const bool lo = X3 && (qs & 2);
        WS_WAIT(&S.b_empty[stage], phase ^ 1u, 0);
        const uint32_t sb = tc::smem_u32(sB + stage * kStageBytes);
        const uint16_t* src;
        int rowlen;
        if (c < nd) {
          src = (lo ? P.fmap_lo : reinterpret_cast<const uint16_t*>(P.fmap)) + c * 64 + q * 8;
          rowlen = P.d;
        } else {
          src = (lo ? P.Gbf_lo : P.Gbf) + (c - nd) * 64 + q * 8;
          rowlen = P.kpadg;
        }
        // rows r0 + kRowStep*j: r & 7 is fixed per thread, so the swizzled destination advances by
        // kRowStep/8 row groups of 1024 bytes per copy
        const uint32_t dst0 = sb + (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + (((q ^ (r0 & 7)) & 7) << 4));
        const long long tl0 = WS_CLOCK();
#pragma unroll
        for (int j = 0; j < kRowsPer; ++j)
          if (rc[j] >= 0) tc::cp_async16(dst0 + (uint32_t)j * (kRowStep / 8 * 1024u), src + (int64_t)rc[j] * rowlen);
        // the stage's full barrier completes when every loader thread's copies have landed (as
        // CUTLASS's SM100 cp.async mainloop: no wait_group, no proxy fence before the UMMA reads)
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&S.b_full[stage]))
                     : "memory");
        if constexpr (PROF) {
          wait_cyc[11] += clock64() - tl0;
          if (warp == 0 && lane == 0) {
            if (pub_group % kCG == kCG - 1) WS_TRACE(pub_tile, 15 + pub_group / kCG);
            if (++pub_group == nstage) { pub_group = 0; ++pub_tile; }
          }
        }
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
      }
      ++t_local;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
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
    int kt_nx = kt_at<LIST>(P, blockIdx.x, nitems);
    for (int64_t tile = blockIdx.x; tile < nitems; tile += gridDim.x) {
      const int kt = kt_nx;
      kt_nx = kt_at<LIST>(P, tile + gridDim.x, nitems);
      bool ok;
      const int ktp = ktp_of(kt, ok, X3 ? kKtX3 : kKtWs);
      if (!ok) continue;
      const int ab = (int)(t_local & 1u);
      WS_WAIT(&S.a_full[ab], (t_local >> 1) & 1u, 1);
      if (lane == 0) WS_TRACE(t_local, 3);
      // the builders wrote A (the tile's bilinear weights) straight into TMEM buffer ab; the MMAs read
      // A from TMEM and B from shared memory; the commit after the last group frees buffer ab
      const uint32_t tA = tA0 + (uint32_t)(ab * (X3 ? kKtX3 / 2 : kKtWs / 2));
      const uint32_t tAlo = tA + (uint32_t)kKtX3;  // x3: lo parts after both hi buffers
      constexpr int gst = X3 ? 2 * kCG : kCG;      // ring stages per MMA group
      tc::fence_after_sync();
      for (int c = 0; c < nch; c += kCG) {
#pragma unroll
        for (int g = 0; g < gst; ++g) WS_WAIT(&S.b_full[stage + g], phase, 2);
        const int db = dcount % kDBufs;
        if (c < nd) WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 3);
        else WS_WAIT(&S.d_empty[db], ((dcount / kDBufs) & 1u) ^ 1u, 4);
        const uint32_t dst = tbase + (uint32_t)(db * kDCols);
        tc::fence_after_sync();
        const long long ti0 = WS_CLOCK();
        {
          // warp-uniform issue (operands in uniform registers, elect.sync picks the issuing lane):
          // one lane under `if (lane == 0)` measured ~100 cycles per MMA, this reaches the 64-cycle
          // tensor rate of M=128, N=128, K=16 (scripts/umma_rate.py)
          const uint32_t b0 = tc::smem_u32(sB + stage * kStageBytes);
          // descriptors advance by 2048 B (start field +128) and 8 TMEM columns per K=16 step
          uint64_t bd = tc::smem_desc_sw128(b0, kStageBytes, 1024);
          uint32_t ta = tA;
          if constexpr (!X3) {
            tc::mma_bf16_ts_elect(dst, ta, bd, idesc, 0u);
#pragma unroll 4
            for (int s = 1; s < ktp / 16; ++s) {
              bd += 128;
              ta += 8;
              tc::mma_bf16_ts_elect(dst, ta, bd, idesc, 1u);
            }
          } else {  // A_hi B_hi + A_hi B_lo + A_lo B_hi (B_lo: the pair's stages + 2)
            uint64_t bl = tc::smem_desc_sw128(b0 + 2 * kStageBytes, kStageBytes, 1024);
            uint32_t tl = tAlo;
            for (int s = 0; s < ktp / 16; ++s) {
              tc::mma_bf16_ts_elect(dst, ta, bd, idesc, s ? 1u : 0u);
              tc::mma_bf16_ts_elect(dst, ta, bl, idesc, 1u);
              tc::mma_bf16_ts_elect(dst, tl, bd, idesc, 1u);
              bd += 128;
              bl += 128;
              ta += 8;
              tl += 8;
            }
          }
#pragma unroll
          for (int g = 0; g < gst; ++g) tc::mma_commit_elect(&S.b_empty[stage + g]);
          tc::mma_commit_elect(&S.d_full[db]);
          if (c + kCG >= nch) tc::mma_commit_elect(&S.a_empty[ab]);
        }
        __syncwarp();
        if constexpr (PROF) issue_cyc += clock64() - ti0;
        if (lane == 0) WS_TRACE(t_local, 4 + c / kCG);
        ++dcount;
        stage += gst;
        if (stage == kStages) { stage = 0; phase ^= 1u; }
      }
      ++t_local;
    }
  } else if (warp < kAccWarp0) {
    reg_dealloc<kRegProducer>();  // idle warp of the second group
  } else if (warp >= kBuildWarp0) {
    // ================= A builders: W straight into TMEM =================
    // Builder warp 16 + j owns TMEM lane group q = j & 3 (tile rows 32q .. 32q + 31; tcgen05.st can
    // only reach a warp's own lane quarter) and every other view present in the tile (rank parity
    // j >> 2). For each of its views it writes all 32 rows' columns of that view's window (zeros
    // where a row does not see the view), so every column of the tile's A is written exactly once.
    // The taps come from a first-order expansion of fu, fv (fusion.py:83-86) around the tile centre
    // (error ~1e-3 px over a tile), clamped into prep's window (a tap can only leave it when its
    // weight is ~0); tiles wider than 2 kAffineR use the exact fp32 projection, bit-identical to
    // prep's (pf_tile_dev.cuh). A 2x2 window (the common case: a tile is ~1/10 of a feature cell)
    // is two TMEM columns written with one tcgen05.st.x2.
    reg_dealloc<kRegProducer>();
    const int bj = warp - kBuildWarp0, bq = bj & 3, bh = bj >> 2, bt = tid - kBuildWarp0 * 32;
    const int row = 32 * bq + lane;
    const uint32_t t_lanes = (uint32_t)(32 * bq) << 16;
    uint32_t t_local = 0;
    static_assert(kMaxViewsTC <= kBuildThreads, "one window per builder thread");
    auto fetch = [&](int64_t t, int& kt, uint2& ds, float4& pp, uint2& mm, int32_t& cd) {
      kt = kt_at<LIST>(P, t, nitems);
      pp = make_float4(0.f, 0.f, 0.f, 0.f);
      mm = make_uint2(0u, 0u);  // rows outside the work item: empty mask
      cd = -1;
      if (t >= nitems) return;
      if (bt < P.nv) ds = P.tile_desc[desc_item<LIST>(P, t) * P.nv + bt];
      int64_t jr;
      if (item_row<LIST>(P, t, ntiles, row, jr)) {
        pp = ld_pref_f4(P.spts + jr);
        const uint4 r4 = ld_pref_u4(P.srec + jr);
        mm = make_uint2(r4.x, r4.y);
        cd = (int32_t)r4.w;
      }
    };
    int kt_nx = 0;
    uint2 ds_nx = make_uint2(0u, 0u), mw_nx;
    float4 p_nx;
    int32_t cd_nx;
    fetch(blockIdx.x, kt_nx, ds_nx, p_nx, mw_nx, cd_nx);
    const float wf1 = (float)(S.sv[0].Wf - 1), hf1 = (float)(S.sv[0].Hf - 1);  // uniform maps (tile_path_ok)
    for (int64_t tile = blockIdx.x; tile < nitems; tile += gridDim.x) {
      const int kt = kt_nx;
      const uint2 ds_cur = ds_nx;
      const float4 p = p_nx;
      const uint2 mw = mw_nx;
      const int32_t cd = cd_nx;
      fetch(tile + gridDim.x, kt_nx, ds_nx, p_nx, mw_nx, cd_nx);
      bool ok;
      const int ktp = ktp_of(kt, ok, X3 ? kKtX3 : kKtWs);
      if (!ok) continue;
      if (bh == 0 && P.vox_list) {
        // touched-voxel list without returning atomics: slot jpt holds the code when this row is the
        // lowest lane of its warp with that code (a warp's sorted points share a few voxels), else
        // -1; pf_voxel_mass_sparse claims each voxel once (atomicExch on its count)
        const uint32_t peers = __match_any_sync(0xffffffffu, cd);
        const bool first = (peers & ((1u << lane) - 1u)) == 0u;
        int64_t jr;
        if (cd >= 0 && item_row<LIST>(P, tile, ntiles, row, jr)) P.vox_list[jr] = first ? cd : -1;
      }
      if (bt == 0) WS_TRACE(t_local, 0);
      const int ab = (int)(t_local & 1u);
      uint2* sdesc = S.desc_a[ab];
      if (bt < P.nv) sdesc[bt] = ds_cur;
      // tile box over the valid rows: expansion point and width (this warp's rows, then all four
      // lane groups through shared memory)
      float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      int64_t jrow;
      if (item_row<LIST>(P, tile, ntiles, row, jrow)) {
        lo[0] = hi[0] = p.x;
        lo[1] = hi[1] = p.y;
        lo[2] = hi[2] = p.z;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
          hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
      if (lane == 0 && bh == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          S.bbox[ab][bq][a] = lo[a];
          S.bbox[ab][bq][a + 3] = hi[a];
        }
      asm volatile("bar.sync 1, %0;" ::"n"(kBuildThreads) : "memory");  // windows + boxes visible
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(fminf(S.bbox[ab][0][a], S.bbox[ab][1][a]), fminf(S.bbox[ab][2][a], S.bbox[ab][3][a]));
        hi[a] = fmaxf(fmaxf(S.bbox[ab][0][a + 3], S.bbox[ab][1][a + 3]), fmaxf(S.bbox[ab][2][a + 3], S.bbox[ab][3][a + 3]));
      }
      const float ox = 0.5f * (lo[0] + hi[0]), oy = 0.5f * (lo[1] + hi[1]), oz = 0.5f * (lo[2] + hi[2]);
      const float ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
      // x3 (fp32 bar): always the exact fp32 projection, as prep's taps
      const bool exact = X3 || ex * ex + ey * ey + ez * ez > 4.f * kAffineR * kAffineR;
      // views with taps in this tile, by rank; coefficients of rank 8 l + bj by lane l of warp bj
      const uint2 dlo = lane < P.nv ? sdesc[lane] : make_uint2(0u, 0u);
      const uint2 dhi = lane + 32 < P.nv ? sdesc[lane + 32] : make_uint2(0u, 0u);
      const uint32_t vm0 = __ballot_sync(0xffffffffu, (dlo.y & 0xffu) != 0u);
      const uint32_t vm1 = __ballot_sync(0xffffffffu, (dhi.y & 0xffu) != 0u);
      const int n0 = __popc(vm0), nvp = n0 + __popc(vm1);
      {
        const int rk = kBuildWarps * lane + bj;
        if (lane < kMaxViewsTC / kBuildWarps && rk < nvp) {
          const int v = rk < n0 ? (int)__fns(vm0, 0, rk + 1) : 32 + (int)__fns(vm1, 0, rk - n0 + 1);
          const float4* vp = S.vpk[v];
          const float4 c0 = vp[0], c1 = vp[1], c2 = vp[2], kk = vp[3], mm = vp[4];
          const float X = fmaf(c0.z, oz, fmaf(c0.y, oy, c0.x * ox)) + c0.w;
          const float Y = fmaf(c1.z, oz, fmaf(c1.y, oy, c1.x * ox)) + c1.w;
          const float Z = fmaf(c2.z, oz, fmaf(c2.y, oy, c2.x * ox)) + c2.w;
          const float rz = 1.f / Z, xr = X * rz, yr = Y * rz;
          const float su = mm.x * kk.x * rz, sv = mm.y * kk.z * rz;  // d fu / d X_cam, d fv / d Y_cam
          const uint2 ds = sdesc[v];
          // the expansion's constant terms are taken relative to the window origin (wx0, wy0)
          S.vcoef[ab][rk][0] = make_float4((fmaf(kk.x, xr, kk.y) + 0.5f) * mm.x - 0.5f - (float)((ds.x >> 16) & 0xff),
                                           su * (c0.x - xr * c2.x), su * (c0.y - xr * c2.y), su * (c0.z - xr * c2.z));
          S.vcoef[ab][rk][1] = make_float4((fmaf(kk.z, yr, kk.w) + 0.5f) * mm.y - 0.5f - (float)(ds.x >> 24),
                                           sv * (c1.x - yr * c2.x), sv * (c1.y - yr * c2.y), sv * (c1.z - yr * c2.z));
          S.vrank[ab][rk] = v | (int)((ds.x & 0xffff) << 8);  // view | window base << 8
          S.vwin[ab][rk] = make_int4((ds.x >> 16) & 0xff, ds.x >> 24, ds.y & 0xff, (ds.y >> 8) & 0xff);
        }
      }
      // this tile's TMEM A buffer is free once the MMAs of the tile two back have completed
      WS_WAIT(&S.a_empty[ab], ((t_local >> 1) & 1u) ^ 1u, 5);
      const long long tb0 = WS_CLOCK();
      asm volatile("bar.sync 1, %0;" ::"n"(kBuildThreads) : "memory");  // coefficients visible
      if (bt == 0) WS_TRACE(t_local, 1);
      tc::fence_after_sync();
      const uint32_t tAb = tA0 + (uint32_t)(ab * (X3 ? kKtX3 / 2 : kKtWs / 2)) + t_lanes;
      constexpr bool x3 = X3;  // lo parts at + kKtX3 columns
      const long long tb1 = WS_CLOCK();
      if constexpr (PROF) wait_cyc[14] += tb1 - tb0;
      const float dxp = p.x - ox, dyp = p.y - oy, dzp = p.z - oz;
      // one view's 32 rows: fast path for 2x2 windows (two TMEM columns), general otherwise;
      // coordinates relative to the window origin
      auto unit_general = [&](int rk) {
        const int vb = S.vrank[ab][rk];
        const int v = vb & 0xff, base = vb >> 8;
        const int4 wn = S.vwin[ab][rk];
        const int wx0 = wn.x, wy0 = wn.y, ww = wn.z, wh = wn.w;
        const bool vis = (((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) != 0u;
        float fu, fv;
        if (!exact) {
          const float4 A0 = S.vcoef[ab][rk][0], A1 = S.vcoef[ab][rk][1];
          fu = fmaf(A0.w, dzp, fmaf(A0.z, dyp, fmaf(A0.y, dxp, A0.x))) + (float)wx0;
          fv = fmaf(A1.w, dzp, fmaf(A1.z, dyp, fmaf(A1.y, dxp, A1.x))) + (float)wy0;
        } else {
          const ProjF pr = project_f32(S.sv[v], p.x, p.y, p.z);
          const TapF tf = taps_f32(S.sv[v], pr.u, pr.v);
          fu = (float)tf.x0 + tf.wx;  // reproduces the clamped coordinate exactly
          fv = (float)tf.y0 + tf.wy;
        }
        const uint32_t col0 = tAb + (uint32_t)(base >> 1);
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
        auto tapw = [&](int k) {
          return vis ? (k == t00 ? w00 : 0.f) + (k == t01 ? w01 : 0.f) + (k == t10 ? w10 : 0.f) + (k == t11 ? w11 : 0.f)
                     : 0.f;
        };
        const int ncols = (ww * wh + 1) >> 1;
        for (int j = 0; j < ncols; ++j) {  // warp-uniform
          const float w0 = tapw(2 * j), w1 = tapw(2 * j + 1);
          const __nv_bfloat162 pr = __floats2bfloat162_rn(w0, w1);
          tc::tmem_st_x1(col0 + (uint32_t)j, *reinterpret_cast<const uint32_t*>(&pr));
          if constexpr (x3) {
            const __nv_bfloat162 pl = __floats2bfloat162_rn(w0 - __low2float(pr), w1 - __high2float(pr));
            tc::tmem_st_x1(col0 + (uint32_t)(kKtX3 + j), *reinterpret_cast<const uint32_t*>(&pl));
          }
        }
      };
      // windows with sides in {2, 3} (~99.5% of them at C5): the row's weights are separable,
      // vx (over the window's columns) x vy (over its rows); clamping into the window reproduces the
      // reference taps (an exact tap can never leave the window; an expanded one only with ~0 weight)
      auto small = [&](auto WWc, auto WHc, int v, int base, float fu_rel, float fv_rel) {
        constexpr int ww = decltype(WWc)::value, wh = decltype(WHc)::value;
        const bool vis = (((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) != 0u;
        const float xr = fminf(fmaxf(fu_rel, 0.f), (float)(ww - 1)), yr = fminf(fmaxf(fv_rel, 0.f), (float)(wh - 1));
        const float ixf = fminf(floorf(xr), (float)(ww - 2)), iyf = fminf(floorf(yr), (float)(wh - 2));
        const float wx = xr - ixf, wy = yr - iyf;
        const float g = vis ? 1.f : 0.f;
        // x weights over 3 columns / y weights over 3 rows (third entry only for width/height 3)
        const bool xa = ixf == 0.f, ya = iyf == 0.f;
        const float vx0 = xa ? 1.f - wx : 0.f, vx1 = xa ? wx : 1.f - wx, vx2 = xa ? 0.f : wx;
        const float vy0 = ya ? g * (1.f - wy) : 0.f, vy1 = ya ? g * wy : g * (1.f - wy), vy2 = ya ? 0.f : g * wy;
        const uint32_t col0 = tAb + (uint32_t)(base >> 1);
        auto pk = [](float lo, float hi) {
          const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
          return *reinterpret_cast<const uint32_t*>(&b2);
        };
        // x3: the bf16 residuals of the same pairs
        auto pkl = [](float lo, float hi) {
          const __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
          const __nv_bfloat162 r2 = __floats2bfloat162_rn(lo - __low2float(b2), hi - __high2float(b2));
          return *reinterpret_cast<const uint32_t*>(&r2);
        };
        auto emit = [&](auto PK, uint32_t c0) {
          if constexpr (ww == 2 && wh == 2) {
            tc::tmem_st_x2(c0, PK(vy0 * vx0, vy0 * vx1), PK(vy1 * vx0, vy1 * vx1));
          } else if constexpr (ww == 3 && wh == 2) {  // taps r0: 0 1 2, r1: 3 4 5
            tc::tmem_st_x2(c0, PK(vy0 * vx0, vy0 * vx1), PK(vy0 * vx2, vy1 * vx0));
            tc::tmem_st_x1(c0 + 2u, PK(vy1 * vx1, vy1 * vx2));
          } else if constexpr (ww == 2 && wh == 3) {  // taps r0: 0 1, r1: 2 3, r2: 4 5
            tc::tmem_st_x2(c0, PK(vy0 * vx0, vy0 * vx1), PK(vy1 * vx0, vy1 * vx1));
            tc::tmem_st_x1(c0 + 2u, PK(vy2 * vx0, vy2 * vx1));
          } else {  // 3 x 3: taps 0..8 + one padding tap
            tc::tmem_st_x4(c0, PK(vy0 * vx0, vy0 * vx1), PK(vy0 * vx2, vy1 * vx0), PK(vy1 * vx1, vy1 * vx2),
                           PK(vy2 * vx0, vy2 * vx1));
            tc::tmem_st_x1(c0 + 4u, PK(vy2 * vx2, 0.f));
          }
        };
        emit(pk, col0);
        if constexpr (x3) emit(pkl, col0 + (uint32_t)kKtX3);
      };
      // rank rk: view, window base and the row's coordinates relative to the window origin
      auto coords = [&](int rk, int& v, int& base, float& fu_rel, float& fv_rel) {
        const int vb = S.vrank[ab][rk];
        v = vb & 0xff;
        base = vb >> 8;
        if (!exact) {
          const float4 A0 = S.vcoef[ab][rk][0], A1 = S.vcoef[ab][rk][1];
          fu_rel = fmaf(A0.w, dzp, fmaf(A0.z, dyp, fmaf(A0.y, dxp, A0.x)));
          fv_rel = fmaf(A1.w, dzp, fmaf(A1.z, dyp, fmaf(A1.y, dxp, A1.x)));
        } else {
          const int4 wn = S.vwin[ab][rk];
          const ProjF pr = project_f32(S.sv[v], p.x, p.y, p.z);
          const TapF tf = taps_f32(S.sv[v], pr.u, pr.v);
          fu_rel = (float)(tf.x0 - wn.x) + tf.wx;
          fv_rel = (float)(tf.y0 - wn.y) + tf.wy;
        }
      };
      // this warp's ranks (bh, bh + 2, ...) grouped by window shape (lane l <-> rank bh + 2 l); two
      // units of one shape are built together: independent chains the scheduler interleaves
      int cls = -1;
      if (lane < ((nvp - bh + 1) >> 1)) {
        const int4 wn = S.vwin[ab][bh + 2 * lane];
        cls = (wn.z == 2 && wn.w == 2)   ? 0
              : (wn.z == 3 && wn.w == 2) ? 1
              : (wn.z == 2 && wn.w == 3) ? 2
              : (wn.z == 3 && wn.w == 3) ? 3
                                         : 4;
      }
      auto run = [&](uint32_t m, auto WWc, auto WHc) {
        while (m) {  // warp-uniform
          int v1, b1, v2, b2;
          float u1, w1, u2, w2;
          coords(bh + 2 * (__ffs(m) - 1), v1, b1, u1, w1);
          m &= m - 1;
          if (m) {
            coords(bh + 2 * (__ffs(m) - 1), v2, b2, u2, w2);
            m &= m - 1;
            small(WWc, WHc, v1, b1, u1, w1);
            small(WWc, WHc, v2, b2, u2, w2);
          } else {
            small(WWc, WHc, v1, b1, u1, w1);
          }
        }
      };
      using I2 = std::integral_constant<int, 2>;
      using I3 = std::integral_constant<int, 3>;
      run(__ballot_sync(0xffffffffu, cls == 0), I2{}, I2{});
      run(__ballot_sync(0xffffffffu, cls == 1), I3{}, I2{});
      run(__ballot_sync(0xffffffffu, cls == 2), I2{}, I3{});
      run(__ballot_sync(0xffffffffu, cls == 3), I3{}, I3{});
      for (uint32_t m = __ballot_sync(0xffffffffu, cls == 4); m; m &= m - 1) unit_general(bh + 2 * (__ffs(m) - 1));
      if (bh == 0)  // columns past the last window (K padding to 16) must be zero too
        for (int j = kt >> 1; j < (ktp >> 1); ++j) {
          tc::tmem_st_x1(tAb + (uint32_t)j, 0u);
          if constexpr (x3) tc::tmem_st_x1(tAb + (uint32_t)(kKtX3 + j), 0u);
        }
      const long long tb2 = WS_CLOCK();
      tc::tmem_st_wait();
      if constexpr (PROF) {
        wait_cyc[12] += tb2 - tb1;
        wait_cyc[13] += clock64() - tb2;
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.a_full[ab]);
      if (bt == 0) WS_TRACE(t_local, 2);
      ++t_local;
    }
  } else {
    // ================= accumulators: two warps per TMEM lane group, split by columns =================
    reg_alloc<kRegAcc>();
    const int need_max = (2.f * (1.05f * __ldg(P.tbound) * P.inv_temp * 1.4426950408889634f) <= 120.f) ? 0 : 1;
    const int half = (warp - kAccWarp0) >> 2;          // 0 / 1
    const int row = 32 * (warp & 3) + lane;            // TMEM lane = tile row
    const uint32_t t_lane = (uint32_t)(32 * (warp & 3)) << 16;
    const int k0 = half * kHalfK;
    uint32_t dcount = 0, a_tile = 0;
    // weight totals (integrate.py:133) of this warp's rows, all tiles: lane l holds materials
    // k0 + l and k0 + 32 + l (each tile's 32 rows are folded in by a warp reduce-scatter)
    float wsum[kHalfK / 32];
#pragma unroll
    for (int q = 0; q < kHalfK / 32; ++q) wsum[q] = 0.f;
    // per-thread integrate partials (<= ~1k tiles per CTA: fp32 accumulation, flushed in fp64)
    float pm_sum = 0.f, pmx = 0.f, pmy = 0.f, pmz = 0.f, featured_n = 0.f, pairs = 0.f;
    const bool outs = OUTS && (P.sims || P.weights);
    const bool p_wide = P.p > 2;
    int kt_nx = kt_at<LIST>(P, blockIdx.x, nitems);
    uint2 rec_nx = make_uint2(0u, 0u);  // record words 2, 3: visible-view count, voxel code
    float4 p_nx = make_float4(0.f, 0.f, 0.f, 0.f);
    int64_t j_nx = 0;
    bool v_nx = blockIdx.x < nitems && item_row<LIST>(P, blockIdx.x, ntiles, row, j_nx);
    if (v_nx) {
      rec_nx = ld_pref_u2(reinterpret_cast<const uint32_t*>(P.srec + j_nx) + 2);
      p_nx = ld_pref_f4(P.spts + j_nx);
    }
    for (int64_t tile = blockIdx.x; tile < nitems; tile += gridDim.x) {
      const int kt = kt_nx;
      const uint2 rec = rec_nx;
      const float4 pcur = p_nx;
      const int64_t jpt = j_nx;
      const bool valid = v_nx;
      kt_nx = kt_at<LIST>(P, tile + gridDim.x, nitems);
      v_nx = tile + gridDim.x < nitems && item_row<LIST>(P, tile + gridDim.x, ntiles, row, j_nx);
      if (v_nx) {
        rec_nx = ld_pref_u2(reinterpret_cast<const uint32_t*>(P.srec + j_nx) + 2);
        p_nx = ld_pref_f4(P.spts + j_nx);
      }
      bool ok;
      ktp_of(kt, ok, X3 ? kKtX3 : kKtWs);
      if (!ok) {  // kt == -1: re-run as sub-tiles; otherwise the points go to the SIMT kernel
        if (kt != -1 && valid && half == 0) P.ovf_list[atomicAdd(P.ovf_count, 1)] = __float_as_int(pcur.w);
        continue;
      }
      if ((warp & 3) == 0 && lane == 0) WS_TRACE(a_tile, 52 + half);
      const int count = (int)rec.x;
      const float invc = count > 0 ? 1.f / (float)count : 0.f;
      const int32_t i = valid ? __float_as_int(pcur.w) : 0;
      float ss0 = 0.f, ss1 = 0.f, ss2 = 0.f, ss3 = 0.f;
      // group g (64 columns) belongs to the warps of parity g & 1: the two warps of a lane group
      // drain alternate groups, so one's tcgen05.ld latency overlaps the other's arithmetic
      for (int c = half; c < nd / kCG; c += 2) {  // c: feature group (kCG chunks)
        const uint32_t gi = dcount + (uint32_t)c;
        const int db = (int)(gi % kDBufs);
        if ((warp & 3) == 0 && lane == 0 && c < 2) WS_TRACE(a_tile, 50 + c);
        WS_WAIT(&S.d_full[db], (gi / kDBufs) & 1u, 6);
        if ((warp & 3) == 0 && lane == 0) WS_TRACE(a_tile, 25 + c);
        tc::fence_after_sync();
#pragma unroll
        for (int g2 = 0; g2 < kCG; ++g2) {  // 64 columns per wait (two x32 loads in flight)
          float v64[64];
          tc::tmem_ld64(tbase + (uint32_t)(db * kDCols + 64 * g2) + t_lane, v64);
#pragma unroll
          for (int gh = 0; gh < 2; ++gh) {
          const int g = 2 * g2 + gh;
          float* v = v64 + 32 * gh;
          if (g == 2 * kCG - 1) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.d_empty[db]);  // data is in registers: release the slot
            if ((warp & 3) == 0 && lane == 0) WS_TRACE(a_tile, 35 + c);
          }
          {
            uint64_t s01 = pk2(ss0, ss1), s23 = pk2(ss2, ss3);
#pragma unroll
            for (int q = 0; q < 32; q += 4) {
              const uint64_t a = pk2(v[q], v[q + 1]), b = pk2(v[q + 2], v[q + 3]);
              s01 = ffma2(a, a, s01);
              s23 = ffma2(b, b, s23);
            }
            up2(s01, ss0, ss1);
            up2(s23, ss2, ss3);
          }
          if (OUTS && P.features && valid) {
            float* dst = P.features + (int64_t)i * P.d + c * kDCols + 32 * g;
#pragma unroll
            for (int q = 0; q < 32; q += 4)
              *reinterpret_cast<float4*>(dst + q) =
                  make_float4(v[q] * invc, v[q + 1] * invc, v[q + 2] * invc, v[q + 3] * invc);
          }
          }
        }
      }
      dcount += (uint32_t)(nd / kCG);
      S.xss[half][row] = (ss0 + ss1) + (ss2 + ss3);
      // ---- epilogue on S (this half's materials) ----------------------------------------------------
      // the similarity columns are the tile's last two groups: materials 64 h .. 64 h + 63 in slot h
      const uint32_t sgi = dcount + (kSGroups == 2 ? (uint32_t)half : 0u);
      const int sslot = (int)(sgi % kDBufs);
      WS_WAIT(&S.d_full[sslot], (sgi / kDBufs) & 1u, 7);
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile, 25 + nd / kCG);
      ++a_tile;
      const uint32_t tS = tbase + (uint32_t)(sslot * kDCols + (kSGroups == 2 ? 0 : k0)) + t_lane;
      tc::fence_after_sync();
      // this half's 64 similarity columns -> registers, then the slot goes straight back to the MMA
      // warp (it moves on to the next tile's feature groups while this epilogue runs)
      float v[kHalfK];
      static_assert(kHalfK == 64, "one tcgen05.ld.x64 per half");
      tc::tmem_ld64(tS, v);
      tc::fence_before_sync();
      asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");  // |F|^2 halves + S reads done
      if (kSGroups == 2) {
        if (lane == 0) mbar_arrive(&S.d_empty[sslot]);  // similarity group h: read by half h only
      } else if (lane == 0 && half == 0) {
        mbar_arrive(&S.d_empty[sslot]);  // both halves have read the group
      }
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile - 1, 45);
      const float ss = S.xss[0][row] + S.xss[1][row];
      const bool featured = valid && count > 0;
      const float inv = ss > 0.f ? rsqrtf(ss) : 0.f;
      const float sc = inv * P.inv_temp * 1.4426950408889634f;  // log2(e) / (T |F|)
      if (outs && P.sims && valid) {  // validation output: cosine similarities, caller's order
#pragma unroll
        for (int q = 0; q < kHalfK; ++q)
          if (k0 + q < P.k) P.sims[(int64_t)i * P.k + k0 + q] = featured ? v[q] * inv : 0.f;
      }
      // exponents are shifted by the constant -c of the setup (yp .z/.w), or by the row max when
      // need_max (grounding.py:175-177); both leave the softmax unchanged up to rounding
      float m2 = 0.f;
      if (need_max) {
        float mx = -INFINITY;
#pragma unroll
        for (int q = 0; q < kHalfK; ++q) {
          const float4 yb = S.yp[2 * ((k0 + q) >> 1) + 1];
          mx = fmaxf(mx, fmaf(v[q], sc, (q & 1) ? yb.w : yb.z));
        }
        S.xm[half][row] = mx;
        asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
        m2 = fmaxf(S.xm[0][row], S.xm[1][row]);
        if (!(m2 > -INFINITY)) m2 = 0.f;
      }
      // pass 1, material pairs (k, k+1): exponentials (in place of S), their sum and the regressions
      float se, pl0, pl1, pl2 = 0.f, pl3 = 0.f, pml;
      {
        uint64_t sep = 0ull, p0p = 0ull, p1p = 0ull, pmp = 0ull;  // (+0.f, +0.f)
        const uint64_t scp = pk2(sc, sc);
#pragma unroll
        for (int q = 0; q < kHalfK; q += 2) {
          // table reads are not hoisted past this point (8 pairs at a time): holding the whole
          // table in registers on top of the 64 S values would push loop state into local memory
          if ((q & 15) == 0) asm volatile("" ::: "memory");
          const int kp = (k0 + q) >> 1;
          const float4 ya = S.yp[2 * kp], yb = S.yp[2 * kp + 1];
          float x0, x1;
          up2(ffma2(pk2(v[q], v[q + 1]), scp, pk2(yb.z - m2, yb.w - m2)), x0, x1);  // padding: -inf
          const float e0 = ex2(x0), e1 = ex2(x1);
          const uint64_t e = pk2(e0, e1);
          sep = fadd2(sep, e);
          p0p = ffma2(e, pk2(ya.x, ya.y), p0p);
          p1p = ffma2(e, pk2(ya.z, ya.w), p1p);
          pmp = ffma2(e, pk2(yb.x, yb.y), pmp);
          v[q] = e0;
          v[q + 1] = e1;
        }
        if (p_wide) {  // regressions 2, 3 (P > 2) from the exponentials, outside the hot loop
#pragma unroll
          for (int q = 0; q < kHalfK; ++q) {
            if ((q & 7) == 0) asm volatile("" ::: "memory");  // table reads not hoisted (registers)
            const float2 y2 = S.yv2[k0 + q];
            pl2 = fmaf(v[q], y2.x, pl2);
            pl3 = fmaf(v[q], y2.y, pl3);
          }
        }
        float a, b;
        up2(sep, a, b);
        se = a + b;
        up2(p0p, a, b);
        pl0 = a + b;
        up2(p1p, a, b);
        pl1 = a + b;
        up2(pmp, a, b);
        pml = a + b;
      }
      S.xsum[half][0][row] = se;
      S.xsum[half][1][row] = pl0;
      S.xsum[half][2][row] = pl1;
      S.xsum[half][3][row] = pl2;
      S.xsum[half][4][row] = pl3;
      S.xsum[half][5][row] = pml;
      asm volatile("bar.sync 2, %0;" ::"n"(kAccThreads) : "memory");
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile - 1, 46);
      const float se_t = S.xsum[0][0][row] + S.xsum[1][0][row];
      // NaN similarity (grounding.py:173-174) -> MaterialError; a non-finite sum otherwise (inf
      // inputs) is flagged too rather than returning NaN properties silently
      if (featured && !(se_t <= 3.4e38f)) atomicOr(P.status, isnan(se_t) ? 1 : 2);
      const float rs = featured ? 1.f / se_t : 0.f;
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile - 1, 47);
      // pass 2: normalised weights of this half -> the warp's weight totals (materials >= K have
      // zero exponentials)
      {
        const uint64_t rsp = pk2(rs, rs);
#pragma unroll
        for (int q = 0; q < kHalfK; q += 2) up2(ffma2(pk2(v[q], v[q + 1]), rsp, 0ull), v[q], v[q + 1]);
      }
      if (outs && P.weights && valid) {  // validation output: softmax weights, caller's order
#pragma unroll
        for (int q = 0; q < kHalfK; ++q)
          if (k0 + q < P.k) P.weights[(int64_t)i * P.k + k0 + q] = v[q];
      }
#pragma unroll
      for (int c = 0; c < kHalfK / 32; ++c) wsum[c] += warp_reduce_scatter32(*reinterpret_cast<float(*)[32]>(v + 32 * c), lane);
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile - 1, 48);
      if (warp == kAccWarp0 && lane == 0) WS_TRACE(a_tile - 1, 49);
      if (warp == kAccWarp0 + 4 && lane == 0) WS_TRACE(a_tile - 1, 54);
      dcount += (uint32_t)kSGroups;
      if (valid && half == 0) {
        float prop[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) prop[pp] = (S.xsum[0][1 + pp][row] + S.xsum[1][1 + pp][row]) * rs;
        const float pm = (S.xsum[0][5][row] + S.xsum[1][5][row]) * rs;
        const float4 p = pcur;
        *(reinterpret_cast<float4*>(P.srec + jpt) + 1) = make_float4(prop[0], prop[1], prop[2], prop[3]);
        if (P.grid_partials && (int32_t)rec.y >= 0) {  // code -1: a padding slot
          const int32_t code = (int32_t)rec.y;
          const int dc = P.density_col;  // selects, not a dynamic index (keeps prop[] in registers)
          const float rho = dc == 0 ? prop[0] : (dc == 1 ? prop[1] : (dc == 2 ? prop[2] : prop[3]));
          atomicAdd(P.grid_partials + code, rho);
          atomicAdd(P.grid_partials + P.cells3 + code, 1.0f);
        }
        const bool live = (int32_t)rec.y >= 0;  // a padding slot (NaN point): no partial contribution
        pm_sum += live ? pm : 0.f;
        pmx = fmaf(live ? pm : 0.f, live ? p.x : 0.f, pmx);
        pmy = fmaf(live ? pm : 0.f, live ? p.y : 0.f, pmy);
        pmz = fmaf(live ? pm : 0.f, live ? p.z : 0.f, pmz);
        featured_n += featured ? 1.f : 0.f;
        pairs += (float)count;
      }
    }
    // flush this CTA's partials (integrate.py:133-155) once
#pragma unroll
    for (int q = 0; q < kHalfK / 32; ++q) {
      const int k = k0 + 32 * q + lane;
      if (k < P.k && wsum[q] != 0.f) atomicAdd(&S.red[k], (double)wsum[q]);
    }
    double r6[6] = {pm_sum, pmx, pmy, pmz, featured_n, pairs};  // fp64 from here on
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
    if (warp == kBuildWarp0) {
      d[12] = (unsigned long long)wait_cyc[12];
      d[13] = (unsigned long long)wait_cyc[13];
      d[14] = (unsigned long long)wait_cyc[14];
    }
  }
#undef WS_WAIT
#undef WS_CLOCK
#undef WS_TRACE
  tc::fence_before_sync();
  __syncthreads();
  if (warp == kAccWarp0) tc::tmem_dealloc(tbase, 512);
}

}  // namespace

int ws_kt_max(bool x3) { return x3 ? kKtX3 : kKtWs; }

size_t ws_smem_bytes() { return (size_t)kStages * kStageBytes + 1024; }

// Launch the persistent kernel (one CTA per SM).
int run_tile_ws(const TileParams& P, cudaStream_t st) {
  if (P.kpadg != kMaxKpadTC) return set_error(PF_ERR_VALUE, "tile_ws: S operand must be %d wide", kMaxKpadTC);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = ws_smem_bytes();
  cudaFuncSetAttribute(k_tile_ws<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_tile_ws<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // (+ sub-tiles, known on the device only; list mode: the list length is on the device too)
  const int64_t ntiles = P.wlist ? (int64_t)sms : (P.n + kTile - 1) / kTile;
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
  static uint32_t* trace = nullptr;
  const char* trace_path = getenv("PF_WS_TRACE");
  if (debug && trace_path) {
    if (!trace) cudaMalloc(&trace, sizeof(uint32_t) * kTraceCtas * kTraceTiles * kTraceEvents);
    cudaMemsetAsync(trace, 0xff, sizeof(uint32_t) * kTraceCtas * kTraceTiles * kTraceEvents, st);
    Q.trace = trace;
  }
  const bool outs = P.sims || P.weights || P.features;
  if (P.wlist) {  // the Gram path's split items (bf16)
    cudaFuncSetAttribute(k_tile_ws<false, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_tile_ws<false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (outs) k_tile_ws<false, true, false, true><<<grid, kWsThreads, smem, st>>>(Q);
    else k_tile_ws<false, false, false, true><<<grid, kWsThreads, smem, st>>>(Q);
    return check_launch("tile_ws_list");
  }
  if (P.x3) {  // f32 maps: the hi / lo split instantiation (the bf16 code is untouched by it)
    if (debug && outs) k_tile_ws<true, true, true><<<grid, kWsThreads, smem, st>>>(Q);
    else if (debug) k_tile_ws<true, false, true><<<grid, kWsThreads, smem, st>>>(Q);
    else if (outs) k_tile_ws<false, true, true><<<grid, kWsThreads, smem, st>>>(Q);
    else k_tile_ws<false, false, true><<<grid, kWsThreads, smem, st>>>(Q);
  } else {
    if (debug && outs) k_tile_ws<true, true, false><<<grid, kWsThreads, smem, st>>>(Q);
    else if (debug) k_tile_ws<true, false, false><<<grid, kWsThreads, smem, st>>>(Q);
    else if (outs) k_tile_ws<false, true, false><<<grid, kWsThreads, smem, st>>>(Q);
    else k_tile_ws<false, false, false><<<grid, kWsThreads, smem, st>>>(Q);
  }
  const int rc = check_launch("tile_ws");
  if (debug && rc == PF_OK) {
    static unsigned long long h[16 * 1024];
    cudaMemcpyAsync(h, dbg, sizeof(unsigned long long) * 16 * grid, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const char* names[15] = {"load:b_empty", "mma:a_full", "mma:b_full", "mma:d_empty(F)", "mma:d_empty(S)",
                             "build:a_empty", "acc:d_full(F)", "acc:d_full(S)", "total", "mma:issue",
                             "load:retire", "load:issue", "build:units", "build:st_wait", "build:coef_bar"};
    fprintf(stderr, "[ws debug] mean cycles per CTA over %d CTAs:", grid);
    for (int q = 0; q < 15; ++q) {
      double sum = 0;
      for (int b = 0; b < grid; ++b) sum += (double)h[b * 16 + q];
      fprintf(stderr, " %s=%.3g", names[q], sum / grid);
    }
    fprintf(stderr, "\n");
    if (trace_path) {
      static uint32_t ht[kTraceCtas * kTraceTiles * kTraceEvents];
      cudaMemcpy(ht, trace, sizeof(ht), cudaMemcpyDeviceToHost);
      if (FILE* f = fopen(trace_path, "wb")) {
        fwrite(ht, sizeof(ht), 1, f);
        fclose(f);
      }
    }
  }
  return rc;
}

}  // namespace tile
}  // namespace pf

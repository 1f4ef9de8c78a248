// Tensor-core tile path of the fused query for bf16 feature maps (BASELINE configs 3 and 5).
//
// Why: the per-point gather F_i = sum_taps w * f_tap reads 4 taps x D channels per visible view; at
// C5 (16M points x 64 views x D=1024) the SIMT kernel moves ~20 GB through L2 and sits at ~250 ms
// (profiles/r01_ncu_c5_simt.txt). Points that are close in space share their taps, so a tile of
// 128 spatially-sorted points needs only ~150 distinct (view, cell) taps. The tile's fused
// features are then a dense contraction  F_tile (128 x D) = W (128 x Kt) . Fmap_taps (Kt x D)
// — the bilinear weights of every point against every tap of its tile (zero where a point does not
// use a tap) — which runs on the 5th-generation tensor cores (tcgen05.mma, bf16 in, fp32 in TMEM).
// The similarity needs only <F_i, t_k> and |F_i| (fusion.py:210-214, grounding.py:158-165):
//   S_tile (128 x K) = W . G_taps,  G = fmap @ text^T (per cell, precomputed),
// and |F_i|^2 from the D-chunks of F_tile drained out of TMEM. Softmax / regression / voxel and
// integrate partials run in the epilogue with one thread per point (grounding.py:168-202,
// integrate.py:133-155).
//
// Kernels (this file; the tensor-core tile kernel is pf_tile_ws.cu):
//   k_sort_keys + CUB DeviceRadixSort::SortPairs + k_sort_gather — stable sort of the points by a
//       21-bit (24-bit from 4M points) Hilbert key of a 128^3 (256^3) grid over the bbox (spatially
//       coherent tiles; the stable sort makes them deterministic);
//   k_tile_prep — per tile: each view is first classified for the box of every 32 points (OFF:
//       occluded or off-image for every point; FULL: visible for every point; MIXED), rigorously,
//       from the box corners and the stored depths under the box's pixel footprint. Only MIXED views get the
//       exact per-point test (fp32 projection with a rigorous error bound, fp64 fallback near any
//       decision boundary -> bit-identical masks). Writes the sorted records (mask, count, voxel
//       code) and each view's tap window of the tile;
//   k_unsort — gathers the sorted records back to the caller's point order.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pf_common.cuh"
#include "pf_tc.cuh"
#include "pf_tile.cuh"

#include <cub/device/device_radix_sort.cuh>
#include "pf_tile_dev.cuh"

namespace pf {
namespace tile {

// ---- counting sort by a coarse space-filling-curve key ------------------------------------------------

// 3-D Hilbert index of a cell of the 2^bits grid: consecutive keys are face-adjacent cells, so a run
// of consecutive sorted points (a tile) stays one compact surface patch far more often than along a
// Morton (Z) curve, which jumps across the object. The curve is Skilling's transpose algorithm
// ("Programming the Hilbert curve", 2004) run as its equivalent 24-state automaton: reading the
// octant o = (x_b, y_b, z_b) of each level from the top, entry = kHilbertFsm[state][o] holds the key
// digit (bits 0-2) and 8 * the next state (bits 3-7); the root state is 0 for every grid order. The
// table was derived from the transpose algorithm and is checked against it on every cell of the
// 2^7 and 2^8 grids (tests/test_oracle.py::TestHilbertKeys via pf_hilbert_table, and on the device
// through pf_hilbert_keys). ~6 instructions per level instead of the transpose's ~35.
constexpr int kHilbertStates = 24;
#define PF_HILBERT_FSM \
      8,  17,  27,   2,  39,  46,  52,   5, \
     56,  71,  73,  86,  91,  20,  10,  13, \
     48,   1, 103, 110, 115,  18,  12,  21, \
    126, 129,  29,  26,  79,  80, 140,   3, \
    148,  43,  37,  34, 127, 128,  78,  81, \
    156,  45,  35,  42,  31,   6, 160, 105, \
     72,  87, 139,   4,  57,  70,  50,  53, \
      0, 171, 111,  76,  49,  58, 102,  61, \
    180, 143,  83, 184,  69,  54,  66,  97, \
     16, 123,   9,  74,  47,  60,  38,  77, \
    132,  95,  85,  14,  67, 144,  82,  33, \
    142,  55, 185,  96,  93, 116,  90,  11, \
    188, 107, 175, 176, 101,  98,  62,  65, \
    164, 109, 119,  22,  99, 106, 152,  41, \
    174, 177,  63,  64, 117, 114,  92,  19, \
     30, 125, 161, 122,   7, 172, 104,  75, \
    130,  25, 133, 166, 179, 136,  84, 191, \
     94,  15, 141,  28, 145,  32, 138,  51, \
    146, 155, 149,  36, 137,  24, 190, 167, \
    154, 157, 147,  44, 169, 182, 120, 135, \
    162, 165, 121, 134, 187, 108, 168, 183, \
    118, 173,  23, 124, 153, 170,  40,  59, \
    178, 113, 131,  88, 181, 158,  68, 151, \
    186, 163,  89, 112, 189, 100, 150, 159,
__constant__ const unsigned char kHilbertFsmC[kHilbertStates * 8] = {PF_HILBERT_FSM};
static const unsigned char kHilbertFsmH[kHilbertStates * 8] = {PF_HILBERT_FSM};  // pf_hilbert_table

// key of the cell (x, y, z) from the table in shared memory (divergent per-lane lookups)
__device__ __forceinline__ uint32_t hilbert_key(const unsigned char* fsm, uint32_t x, uint32_t y, uint32_t z,
                                                int bits) {
  uint32_t key = 0u, s8 = 0u;
#pragma unroll
  for (int b = 7; b >= 0; --b) {
    if (b >= bits) continue;
    const uint32_t o = (((x >> b) & 1u) << 2) | (((y >> b) & 1u) << 1) | ((z >> b) & 1u);
    const uint32_t e = fsm[s8 | o];
    key = (key << 3) | (e & 7u);
    s8 = e & ~7u;
  }
  return key;
}

template <int BITS>  // compile-time grid order: the level loop fully unrolled
__global__ void k_sort_keys(const float* __restrict__ p, int64_t n, const double* __restrict__ lo_hi,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ hist, uint32_t* __restrict__ iota) {
  __shared__ unsigned char fsm[kHilbertStates * 8];
  for (int j = threadIdx.x; j < kHilbertStates * 8; j += blockDim.x) fsm[j] = kHilbertFsmC[j];
  __syncthreads();
  constexpr int cells = 1 << BITS;
  const float lx = (float)lo_hi[0], ly = (float)lo_hi[1], lz = (float)lo_hi[2];
  const float ext = fmaxf(fmaxf((float)(lo_hi[3] - lo_hi[0]), (float)(lo_hi[4] - lo_hi[1])),
                          (float)(lo_hi[5] - lo_hi[2]));
  const float inv = ext > 0.f ? (float)cells / ext : 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int cx = min(max((int)((__ldg(p + 3 * i) - lx) * inv), 0), cells - 1);
    const int cy = min(max((int)((__ldg(p + 3 * i + 1) - ly) * inv), 0), cells - 1);
    const int cz = min(max((int)((__ldg(p + 3 * i + 2) - lz) * inv), 0), cells - 1);
    const uint32_t key = hilbert_key(fsm, (uint32_t)cx, (uint32_t)cy, (uint32_t)cz, BITS);
    if (keys) keys[i] = key;
    if (hist) atomicAdd(hist + key, 1u);
    if (iota) iota[i] = (uint32_t)i;
  }
}

__global__ void k_sort_scatter(const float* __restrict__ p, int64_t n, const uint32_t* __restrict__ keys,
                               uint32_t* __restrict__ cursor, const uint32_t* __restrict__ block_base,
                               int32_t* __restrict__ inv, float4* __restrict__ spts) {
  // one scattered 16-byte write per point (the sorted point carries its original index in .w);
  // the inverse permutation is written coalesced
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = keys[i];
    const uint32_t pos = atomicAdd(cursor + key, 1u) + __ldg(block_base + (key >> 12));
    inv[i] = (int32_t)pos;
    spts[pos] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2),
                            __int_as_float((int32_t)i));
  }
}

// sorted (key, index) pairs -> sorted points carrying their original index, inverse permutation
__global__ void k_sort_gather(const float* __restrict__ p, int64_t n, const uint32_t* __restrict__ idx,
                              int32_t* __restrict__ inv, float4* __restrict__ spts) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[j];
    spts[j] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2), __int_as_float((int32_t)i));
    inv[i] = (int32_t)j;
  }
}

// exclusive scan of the sort's counters: per-block scan of 4096 (1024 threads x 4), block totals,
// then add. In place on `hist`.
__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t* __restrict__ hist, uint32_t* __restrict__ totals) {
  __shared__ uint32_t warp_sums[32];
  const int64_t base = (int64_t)blockIdx.x * 4096 + threadIdx.x * 4;
  uint4 v = *reinterpret_cast<const uint4*>(hist + base);
  const uint32_t s0 = v.x, s1 = s0 + v.y, s2 = s1 + v.z, s3 = s2 + v.w;
  uint32_t incl = s3;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t ws = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += t;
    }
    warp_sums[lane] = ws;
  }
  __syncthreads();
  const uint32_t excl = incl - s3 + (wid > 0 ? warp_sums[wid - 1] : 0u);
  *reinterpret_cast<uint4*>(hist + base) = make_uint4(excl, excl + s0, excl + s1, excl + s2);
  if (threadIdx.x == 1023) totals[blockIdx.x] = excl + s3;
}

__global__ void __launch_bounds__(1024) k_scan_totals(uint32_t* __restrict__ totals, int nblocks) {
  // exclusive scan of <= 4096 block totals, 4 consecutive per thread
  __shared__ uint32_t s[1024];
  const int t = threadIdx.x;
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = 4 * t + q < nblocks ? totals[4 * t + q] : 0u;
    sum += v[q];
  }
  s[t] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t x = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += x;
    __syncthreads();
  }
  uint32_t run = s[t] - sum;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (4 * t + q < nblocks) totals[4 * t + q] = run;
    run += v[q];
  }
}

__global__ void k_scan_add(uint32_t* __restrict__ hist, const uint32_t* __restrict__ totals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  hist[i] += totals[i / 4096];
}

// Per-view constant error bounds over the object's bbox (all points lie inside it): the camera
// coordinates are affine in p, so their extremes over the box are attained at its corners. When
// the whole box is safely in front of the camera the per-sample bound of classify() is replaced by
// one constant per view (same formulas with the worst-case |X|, |Y|, 1/z), which removes the
// per-sample bound arithmetic from the hot loop.
__device__ float4 view_bound(const ViewF& w, const pf_view_t& v, const double* lo_hi) {
  double zmin = 1e300, xmax = 0.0, ymax = 0.0, p1 = 0.0;
  for (int c = 0; c < 8; ++c) {
    const double px = (c & 1) ? lo_hi[3] : lo_hi[0];
    const double py = (c & 2) ? lo_hi[4] : lo_hi[1];
    const double pz = (c & 4) ? lo_hi[5] : lo_hi[2];
    const double X = v.R[0] * px + v.R[1] * py + v.R[2] * pz + v.t[0];
    const double Y = v.R[3] * px + v.R[4] * py + v.R[5] * pz + v.t[1];
    const double Z = v.R[6] * px + v.R[7] * py + v.R[8] * pz + v.t[2];
    zmin = fmin(zmin, Z);
    xmax = fmax(xmax, fabs(X));
    ymax = fmax(ymax, fabs(Y));
    p1 = fmax(p1, fabs(px) + fabs(py) + fabs(pz));
  }
  const double e = (p1 + (double)w.tmax) * 4.76837158203125e-07 * 1.001;  // project_f32's e, maxed
  if (!(zmin > 8.0 * e)) return make_float4(0.f, 0.f, 0.f, 0.f);
  const double zl = zmin - e;  // lower bound of |z| as computed in fp32
  auto err = [&](double f, double c, double num) {
    const double a = (num + e) / zl;
    const double da = e / zl + 2.0 * e * (num + e) / (zl * zl) + 1.2e-7 * a;
    return fabs(f) * da + 1.2e-7 * (fabs(f) * a + fabs(c)) + 1e-6;
  };
  const double eu = err(w.fx, w.cx, xmax), ev = err(w.fy, w.cy, ymax);
  if (eu >= 0.25 || ev >= 0.25) return make_float4(0.f, 0.f, 0.f, 0.f);
  return make_float4((float)(eu * 1.001), (float)(ev * 1.001), (float)e, 1.f);
}

// classify() with the per-view constant bounds (z > 0 and finite u, v are guaranteed)
__device__ __forceinline__ int classify_fast(const ViewF& w, const float4& b, const ProjF& q,
                                             int64_t& didx) {
  const float du = fabsf(q.u - floorf(q.u) - 0.5f), dv = fabsf(q.v - floorf(q.v) - 0.5f);
  if (du <= b.x || dv <= b.y) return kAmbiguous;
  const float ru = rintf(q.u), rv = rintf(q.v);
  if (!(ru >= 0.f && ru < (float)w.W && rv >= 0.f && rv < (float)w.H)) return kInvisible;
  didx = w.depth_off + (int64_t)rv * w.W + (int64_t)ru;
  return kNeedDepth;
}

// ---- tile x view classification ----------------------------------------------------------------------
enum : int { kViewOff = 0, kViewFull = 1, kViewMixed = 2, kViewExact = 3 };
constexpr int kScanMax = 64;  // pixels of depth scanned per (tile, view) at most

// Per-(tile, view) second-order model of a MIXED view (see classify_tile_view), 7 x 16 B read by
// every point of the tile as broadcast shared-memory loads: u, v from a = R0.d, c = R1.d, b = R2.d
// (d = p - o) with rigorous bounds eu, ev, ez on |model - numpy's fp64 value| over the tile box.
struct MixModel {
  float4 ra;  // {R00, R01, R02, u0}
  float4 rc;  // {R10, R11, R12, v0}
  float4 rb;  // {R20, R21, R22, z0}
  float4 cu;  // u = b (qu b + ku a + kb) + (su a + u0): {su, kb, ku, qu}
  float4 cv;  // v = b (qv b + kv c + kc) + (sv c + v0): {sv, kc, kv, qv}
  float4 e;   // {0.5 - eu, 0.5 - ev (rounded down), ez, box window (packed bytes, MIXED -> seen)}
  int2 wh;    // depth map W, H
  const float* dmap;  // this view's depth map
};
static_assert(sizeof(MixModel) == 112, "7 x 16 B");

// Decide one view for every point of a tile at once. The points lie in the box [lo, hi] (exact:
// min / max of their f32 coordinates). Camera coordinates are affine in p, so the camera depth over
// the box lies in [zmin, zmax] of its corners; with the box in front of the camera the pixel
// coordinates u = fx X/Z + cx are linear-fractional, so over the box they lie between the corners'
// extremes. rint is monotone, so every point's depth-map pixel lies in [rint(umin), rint(umax)] x
// [rint(vmin), rint(vmax)] (corner values in fp32 widened by 0.01 px; their fp32 error is < 1e-3
// px). Then, with 1e-5 m slack on every depth comparison (fp32 corner depths are within 1e-6 m):
//   OFF  : the rectangle misses the image, or zmin > (max stored depth in it) + eps for all pixels
//          -> no point passes z <= stored + eps (numpy_impl.py:31-40);
//   FULL : the rectangle is inside the image, every stored depth in it is > 0 and
//          zmax < (min stored depth) + eps -> every point passes;
//   MIXED: per-point test against the affine model (below);
//   EXACT: the box reaches the camera plane or covers > kScanMax pixels: per-point exact test.
// FULL and MIXED views get the box's tap window: fu = (u + 0.5) * Wf/W - 0.5 computed by the same
// monotone fp32 ops as taps_f32 on the widened pixel range bounds every point's taps.
//
// MIXED model: o = box centre, d = p - o, |d| <= r. z is affine in p, so z = Z(o) + R2 . d exactly;
// u = fx X/Z + cx with X = X(o) + a, Z = Z(o) + b (a = R0 . d, b = R2 . d, |a|, |b| <= r):
//   X/Z - [X0/Z0 + a/Z0 - X0 b/Z0^2] = b (X0 b - a Z0) / (Z0^2 Z)
// so the first-order model is within fx r^2 (|X0| + Z0) / (Z0^2 zmin) of the exact value. On top:
// the fp32 error of u(o) (the view's constant project_f32 bound), 3 fma roundings of a ~|u| value
// and the gradient's relative error.
// 1 / z for z > 1e-3 without the fp64 division subroutine: fp32 seed + two Newton steps (a few
// fp64 ulps; the model's bounds allow ~1e-13)
__device__ __forceinline__ double rcp_f64(double z) {
  double r = (double)__frcp_rn((float)z);
  r = fma(r, fma(-z, r, 1.0), r);
  return fma(r, fma(-z, r, 1.0), r);
}

// Two threads per view (lanes 2j, 2j + 1 of a warp: `h` = 0 / 1, `pm` = the pair's lane mask) share
// the work: corners with z = lo / hi, alternate rows of the depth scan, and the u / v halves of the
// MIXED model; shuffles combine them, so both threads take the same decision. The MIXED model is
// written straight into `aff` (shared memory).
__device__ __forceinline__ float pair_min(unsigned pm, float x) { return fminf(x, __shfl_xor_sync(pm, x, 1)); }
__device__ __forceinline__ float pair_max(unsigned pm, float x) { return fmaxf(x, __shfl_xor_sync(pm, x, 1)); }

__device__ __forceinline__ int classify_tile_view(const ViewF& v, const float4& vb, const pf_view_t& v64,
                                                  const float* __restrict__ depth, const float* lo, const float* hi,
                                                  float eps, int h, unsigned pm, bool store, int4& win,
                                                  MixModel& aff) {
  float zmin = 1e30f, zmax = -1e30f, umin = 1e30f, umax = -1e30f, vmin = 1e30f, vmax = -1e30f;
  {
    const float pz = h ? hi[2] : lo[2];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float px = (c & 1) ? hi[0] : lo[0];
      const float py = (c & 2) ? hi[1] : lo[1];
      const float X = fmaf(v.R[2], pz, fmaf(v.R[1], py, v.R[0] * px)) + v.t[0];
      const float Y = fmaf(v.R[5], pz, fmaf(v.R[4], py, v.R[3] * px)) + v.t[1];
      const float Z = fmaf(v.R[8], pz, fmaf(v.R[7], py, v.R[6] * px)) + v.t[2];
      zmin = fminf(zmin, Z);
      zmax = fmaxf(zmax, Z);
      const float rz = __frcp_rn(Z);  // (the 0.01 px widening below covers the fp32 corner error)
      const float u = fmaf(v.fx, X * rz, v.cx), w = fmaf(v.fy, Y * rz, v.cy);
      umin = fminf(umin, u);
      umax = fmaxf(umax, u);
      vmin = fminf(vmin, w);
      vmax = fmaxf(vmax, w);
    }
  }
  zmin = pair_min(pm, zmin);
  zmax = pair_max(pm, zmax);
  umin = pair_min(pm, umin);
  umax = pair_max(pm, umax);
  vmin = pair_min(pm, vmin);
  vmax = pair_max(pm, vmax);
  if (!(zmin > 1e-3f)) return kViewExact;  // the box reaches the camera plane
  const float ulo = fmaxf(umin - 0.01f, -1e6f), uhi = fminf(umax + 0.01f, 1e6f);
  const float vlo = fmaxf(vmin - 0.01f, -1e6f), vhi = fminf(vmax + 0.01f, 1e6f);
  const int x0 = (int)rintf(ulo), x1 = (int)rintf(uhi), y0 = (int)rintf(vlo), y1 = (int)rintf(vhi);
  const int cx0 = max(x0, 0), cx1 = min(x1, v.W - 1), cy0 = max(y0, 0), cy1 = min(y1, v.H - 1);
  if (cx1 < cx0 || cy1 < cy0) return kViewOff;
  const int bw = cx1 - cx0 + 1, bh = cy1 - cy0 + 1;
  if (bw * bh > kScanMax) return kViewExact;
  float dmax = 0.f, dmin = 1e30f;
  {
    const float* d = depth + v.depth_off + (int64_t)(cy0 + h) * v.W + cx0;
    for (int y = h; y < bh; y += 2, d += 2 * v.W)
      for (int x = 0; x < bw; x += 2) {  // two independent loads per step
        const float s0 = __ldg(d + x), s1 = __ldg(d + min(x + 1, bw - 1));
        dmax = fmaxf(dmax, fmaxf(s0, s1));
        dmin = fminf(dmin, fminf(s0, s1));
      }
  }
  dmax = pair_max(pm, dmax);
  dmin = pair_min(pm, dmin);
  if (zmin - 1e-5f > dmax + eps + 1e-5f) return kViewOff;
  // tap window of every point (taps_f32 on the widened range; fu is monotone in u)
  const float fu0 = __fsub_rn(__fmul_rn(__fadd_rn(ulo, 0.5f), v.ru), 0.5f);
  const float fu1 = __fsub_rn(__fmul_rn(__fadd_rn(uhi, 0.5f), v.ru), 0.5f);
  const float fv0 = __fsub_rn(__fmul_rn(__fadd_rn(vlo, 0.5f), v.rv), 0.5f);
  const float fv1 = __fsub_rn(__fmul_rn(__fadd_rn(vhi, 0.5f), v.rv), 0.5f);
  const float wmax = (float)(v.Wf - 1), hmax = (float)(v.Hf - 1);
  win.x = (int)floorf(fminf(fmaxf(fu0, 0.f), wmax));
  win.y = (int)floorf(fminf(fmaxf(fv0, 0.f), hmax));
  win.z = min((int)floorf(fminf(fmaxf(fu1, 0.f), wmax)) + 1, v.Wf - 1);
  win.w = min((int)floorf(fminf(fmaxf(fv1, 0.f), hmax)) + 1, v.Hf - 1);
  const bool inside = x0 >= 0 && y0 >= 0 && x1 < v.W && y1 < v.H;
  if (inside && dmin > 0.f && zmax + 2e-5f < dmin + eps) return kViewFull;
  if (!(vb.w > 0.f)) return kViewExact;  // no constant fp32 bound for this view
  // MIXED: second-order model around the box centre
  const float ox = 0.5f * (lo[0] + hi[0]), oy = 0.5f * (lo[1] + hi[1]), oz = 0.5f * (lo[2] + hi[2]);
  const float hx = 0.5f * (hi[0] - lo[0]), hy = 0.5f * (hi[1] - lo[1]), hz = 0.5f * (hi[2] - lo[2]);
  const float r = sqrtf(hx * hx + hy * hy + hz * hz) * 1.0001f + 1e-7f;
  // the model's value at o in fp64 with the reference's camera: |u0 - u64(o)| is only the final
  // rounding to fp32 (+ ~1e-13), so no fp32 projection bound enters. Thread h builds the u (h = 0)
  // or the v (h = 1) half: W0 = X0 or Y0, f = fx or fy, ...
  const double Z0 = cam_row(v64.R, 2, ox, oy, oz, v64.t[2]);
  const double W0 = cam_row(v64.R, h, ox, oy, oz, v64.t[h]);
  const double f = h ? v64.fy : v64.fx, cc = h ? v64.cy : v64.cx;
  const double rz0 = rcp_f64(Z0);
  const float w0 = (float)fma(f * W0, rz0, cc);
  // second-order model in a = R0.d (c = R1.d for v), b = R2.d (d = p - o):
  //   X/Z = X0/Z0 + a/Z0 - X0 b/Z0^2 - a b/Z0^2 + X0 b^2/Z0^3 + R3,
  //   R3 = a b^2/Z0^3 - (X0 + a) b^3 / (Z0^3 Z),  |R3| <= r^3 ((|X0| + r)/(Z0^3 zmin) + 1/Z0^3)
  const double sw = f * rz0, wr = W0 * rz0;
  const double rr = (double)r;
  const double r3 = rr * rr * rr * (rz0 * rz0 * rz0);  // the bound carries a 1.05 factor
  const double rzl = rcp_f64((double)zmin);
  const double gw = fabs(sw) * (1.0 + fabs(wr)) * rr;                 // |linear part|
  const double qw = fabs(sw) * rz0 * (1.0 + fabs(wr)) * rr * rr;      // |quadratic part|
  // remainder + fp32 rounding of w0 and of the ~6 rounded ops of the evaluation + the fp32 coefficients
  const double ew = fabs(f) * r3 * ((fabs(W0) + rr) * rzl + 1.0) * 1.05 + 7e-7 * (fabs(w0) + gw + qw) +
                    1e-5 * (gw + qw) + 1e-5;
  const bool ok = ew < 0.25;
  // both lanes must reach the shuffle: a short-circuit `ok && shfl(...)` would leave the partner of a
  // lane with ok == false waiting forever
  const bool ok_pair = __shfl_xor_sync(pm, ok, 1);
  if (!(ok && ok_pair)) return kViewExact;
  const float4 row = h ? make_float4(v.R[3], v.R[4], v.R[5], w0) : make_float4(v.R[0], v.R[1], v.R[2], w0);
  const float4 co = make_float4((float)sw, (float)(-sw * wr), (float)(-sw * rz0), (float)(sw * wr * rz0));
  const float hw = __fsub_rd(0.5f, __double2float_ru(ew));
  if (!store) {
  } else if (h == 0) {
    aff.ra = row;
    aff.cu = co;
    aff.e.x = hw;
    aff.rb = make_float4(v.R[6], v.R[7], v.R[8], (float)Z0);
    // z = z0 + b is exactly affine: rounding only; + the 1e-9 floor and the margin / difference roundings
    aff.e.z = (4.7e-7f * (fabsf((float)Z0) + 2.f * r) + 1e-7f) * 1.0001f + 2e-9f;
    aff.wh = make_int2(v.W, v.H);
    aff.dmap = depth + v.depth_off;
  } else {
    aff.rc = row;
    aff.cv = co;
    aff.e.y = hw;
  }
  return kViewMixed;
}

__global__ void k_view_setup(TileParams P) {
  const int j = threadIdx.x;
  if (j < P.nv) {
    const ViewF w = make_viewf(P.views[j], P.d);
    P.viewf[j] = w;
    P.vbound[j] = view_bound(w, P.views[j], P.lo_hi);
  }
  if (j == 0) {  // voxel domain once (the fp64 edge division of voxel_edge)
    double lo[3];
    const double edge = voxel_edge(P.lo_hi, P.grid, lo);
    P.vox[0] = lo[0];
    P.vox[1] = lo[1];
    P.vox[2] = lo[2];
    P.vox[3] = edge;
    float* f = reinterpret_cast<float*>(P.vox + 4);
    f[0] = (float)lo[0];
    f[1] = (float)lo[1];
    f[2] = (float)lo[2];
    f[3] = edge > 0.0 ? (float)(1.0 / edge) : 0.f;
  }
}

// voxel_code (pf_common.cuh, sampling.py:110-123 convention) with an fp32 fast path: q = (p - lo) /
// edge in fp32 is within g * 4e-7 of the fp64 quotient (|p - lo| exact to 2^-24, one rounded 1/edge
// and one product); when every axis is > 1e-3 from an integer its floor equals the fp64 one, else
// the exact fp64 formula decides (~0.6 % of points).
__device__ __forceinline__ int32_t voxel_code_fast(const float4& p, const double* __restrict__ vox, int g) {
  const float* f = reinterpret_cast<const float*>(vox + 4);
  const float inv = f[3];
  const float q[3] = {(p.x - f[0]) * inv, (p.y - f[1]) * inv, (p.z - f[2]) * inv};
  bool ok = inv > 0.f;
  int c[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float fl = floorf(q[a]);
    const float fr = q[a] - fl;
    ok = ok && fr > 1e-3f && fr < 1.f - 1e-3f;
    c[a] = min(max((int)fl, 0), g - 1);
  }
  if (ok) return (c[0] * g + c[1]) * g + c[2];
  const double lo[3] = {vox[0], vox[1], vox[2]};
  return voxel_code(p.x, p.y, p.z, lo, vox[3], g);
}

// exact per-point decision for one (point, view) sample; fills the taps when visible
__device__ __forceinline__ bool point_visible(const ViewF& v, const float4& b, const pf_view_t& v64,
                                              const float* __restrict__ depth, const float4& p,
                                              double eps, float eps_f, TapF& t) {
  const ProjF q = project_f32(v, p.x, p.y, p.z);
  int64_t didx = 0;
  int s = b.w > 0.f ? classify_fast(v, b, q, didx) : classify(v, q, didx);
  if (s == kNeedDepth) s = depth_decide(q, __ldg(depth + didx), eps_f);
  bool vis = s == kNeedDepth;
  if (s == kAmbiguous) vis = visible_f64(v64, depth, p.x, p.y, p.z, eps);  // rare
  if (vis) t = taps_f32(v, q.u, q.v);
  return vis;
}

// MIXED-view decision through the second-order model, branch-free: vis = visible for sure; amb =
// within the model's bound of a pixel boundary or of the depth threshold (the caller re-tests those
// samples exactly). Otherwise invisible (off-image, empty pixel, or behind the stored depth).
__device__ __forceinline__ void affine_visible(const MixModel& m, float dx, float dy, float dz, float eps_f, bool& vis,
                                               bool& amb) {
  const float a = fmaf(m.ra.z, dz, fmaf(m.ra.y, dy, m.ra.x * dx));
  const float c = fmaf(m.rc.z, dz, fmaf(m.rc.y, dy, m.rc.x * dx));
  const float b = fmaf(m.rb.z, dz, fmaf(m.rb.y, dy, m.rb.x * dx));
  const float u = fmaf(b, fmaf(m.cu.w, b, fmaf(m.cu.z, a, m.cu.y)), fmaf(m.cu.x, a, m.ra.w));
  const float v = fmaf(b, fmaf(m.cv.w, b, fmaf(m.cv.z, c, m.cv.y)), fmaf(m.cv.x, c, m.rc.w));
  // |u - rint(u)| (exact in fp32) >= 0.5 - eu  <=>  u within eu of a pixel boundary (bitwise ops: no
  // short-circuit branches)
  const float ru = rintf(u), rv = rintf(v);
  const bool amb_uv = (fabsf(u - ru) >= m.e.x) | (fabsf(v - rv) >= m.e.y);
  // one unsigned compare per axis (finite u, v: the model of finite points)
  const int iu = (int)ru, iv = (int)rv;
  const bool inb = ((unsigned)iu < (unsigned)m.wh.x) & ((unsigned)iv < (unsigned)m.wh.y) & !amb_uv;
  float stored = 0.f;
  if (inb) stored = __ldg(m.dmap + (iv * m.wh.x + iu));  // a view's map has < 2^31 pixels
  const float thr = __fadd_rn(stored, eps_f);  // > 0 when stored > 0
  const float mz = fmaf(2.4e-7f, thr, m.e.z);  // m.e.z includes the 1e-9 floor
  const float dz_ = (m.rb.w + b) - thr;
  const bool hit = stored > 0.f;               // (inb folded in: stored = 0 otherwise)
  const bool near = dz_ < -mz;                 // z + mz < thr, up to the margin's own rounding slack
  vis = hit & near;
  amb = amb_uv | (hit & !near & !(dz_ > mz));
}

// ---- k_tile_prep ---------------------------------------------------------------------------------------
__device__ __forceinline__ void window_reduce(bool vis, const TapF& t, int* wx0, int* wy0, int* wx1, int* wy1,
                                              int v, int lane) {
  if (__any_sync(0xffffffffu, vis)) {
    const int ax0 = __reduce_min_sync(0xffffffffu, vis ? t.x0 : INT_MAX);
    const int ay0 = __reduce_min_sync(0xffffffffu, vis ? t.y0 : INT_MAX);
    const int ax1 = __reduce_max_sync(0xffffffffu, vis ? t.x0 + t.dx : -1);
    const int ay1 = __reduce_max_sync(0xffffffffu, vis ? t.y0 + t.dy : -1);
    if (lane == 0) {
      atomicMin(wx0 + v, ax0);
      atomicMin(wy0 + v, ay0);
      atomicMax(wx1 + v, ax1);
      atomicMax(wy1 + v, ay1);
    }
  }
}

// TR = rows per tile (128: k_tile_ws; kGramTile: the Gram kernel), one thread per point
template <int TR>
__global__ void __launch_bounds__(TR, TR == kTile ? 8 : 2) k_tile_prep(TileParams P) {
  __shared__ ViewF sv[kMaxViewsTC];
  __shared__ MixModel saff[kMaxViewsTC];
  __shared__ float4 sbound[kMaxViewsTC];
  __shared__ int wx0[kMaxViewsTC], wx1[kMaxViewsTC], wy0[kMaxViewsTC], wy1[kMaxViewsTC];
  __shared__ unsigned char s_cls[kMaxViewsTC];
  __shared__ unsigned char s_list[kMaxViewsTC];  // MIXED views, then EXACT views
  __shared__ uint32_t s_full[2], s_seen[2];
  __shared__ int s_nmixed, s_nexact;
  __shared__ float sbb[TR / 32][6];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t tile = blockIdx.x;
  const int64_t jpt = tile * TR + tid;
  const bool valid = jpt < P.n;
  const float4 p = valid ? P.spts[jpt] : make_float4(0.f, 0.f, 0.f, 0.f);
  const bool live = valid && !isnan(p.x);  // NaN point: a padding slot (pf_shard_pack_padded)
  {
    const bool inbox = live && !isnan(p.y) && !isnan(p.z);
    // tile box: warp min / max as order-preserving integer reductions (one REDUX each); rows past n
    // and padding slots contribute nothing
    const int b[6] = {__reduce_min_sync(0xffffffffu, float_key(inbox ? p.x : INFINITY)),
                      __reduce_min_sync(0xffffffffu, float_key(inbox ? p.y : INFINITY)),
                      __reduce_min_sync(0xffffffffu, float_key(inbox ? p.z : INFINITY)),
                      __reduce_max_sync(0xffffffffu, float_key(inbox ? p.x : -INFINITY)),
                      __reduce_max_sync(0xffffffffu, float_key(inbox ? p.y : -INFINITY)),
                      __reduce_max_sync(0xffffffffu, float_key(inbox ? p.z : -INFINITY))};
    if (lane == 0)
#pragma unroll
      for (int a = 0; a < 6; ++a) sbb[tid >> 5][a] = key_float(b[a]);
  }
  if (tid < 2) s_seen[tid] = 0u;
  __syncthreads();
  float lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = sbb[0][a];
    hi[a] = sbb[0][a + 3];
#pragma unroll
    for (int w = 1; w < TR / 32; ++w) {
      lo[a] = fminf(lo[a], sbb[w][a]);
      hi[a] = fmaxf(hi[a], sbb[w][a + 3]);
    }
  }
  const float eps_f = (float)P.eps;
  if (P.tbox && tid == 0) {
    P.tbox[2 * tile] = make_float4(lo[0], lo[1], lo[2], 0.f);
    P.tbox[2 * tile + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
  }
  {
    // two threads per view; every thread runs (a view index past nv repeats the last view and writes
    // nothing), so the pair shuffles always see both lanes
    const int cv = tid >> 1, h = tid & 1;
    const int vj = min(cv, P.nv - 1);
    const unsigned pm = 3u << (lane & 30);
    const ViewF v = P.viewf[vj];  // per-view fp32 camera + constant error bounds (k_view_setup)
    const float4 vb = P.vbound[vj];
    int4 win = make_int4(INT_MAX, INT_MAX, -1, -1);
    const bool mine = cv < P.nv;
    const int cls = classify_tile_view(v, vb, P.views[vj], P.depth, lo, hi, eps_f, h, pm, mine, win, saff[vj]);
    if (mine && h == 0) {
      s_cls[cv] = (unsigned char)cls;
      // FULL: box window now; MIXED: box window once a point is seen visible; EXACT: per-point union
      const bool boxwin = cls == kViewFull;
      wx0[cv] = boxwin ? win.x : INT_MAX;
      wy0[cv] = boxwin ? win.y : INT_MAX;
      wx1[cv] = boxwin ? win.z : -1;
      wy1[cv] = boxwin ? win.w : -1;
      if (cls == kViewMixed || cls == kViewExact) {  // (re-read: keeps v out of the live range)
        sv[cv] = P.viewf[cv];
        sbound[cv] = P.vbound[cv];
      }
      // stash the MIXED box window in the model's spare slot until visibility is known
      if (cls == kViewMixed) saff[cv].e.w = __int_as_float(win.x | (win.y << 8) | (win.z << 16) | (win.w << 24));
      if (P.dbg && cls == kViewMixed) {  // mean eu of the models
        atomicAdd(P.dbg + 16 * 1000 + 9, (unsigned long long)((0.5f - saff[cv].e.x) * 1e6f));
        atomicAdd(P.dbg + 16 * 1000 + 10, 1ull);
      }
    }
  }
  __syncthreads();
  if (tid < 32) {  // ballot compaction: FULL bitmask, MIXED then EXACT list (<= 64 views: two per lane)
    const bool m0 = lane < P.nv && s_cls[lane] == kViewMixed;
    const bool m1 = lane + 32 < P.nv && s_cls[lane + 32] == kViewMixed;
    const bool e0 = lane < P.nv && s_cls[lane] == kViewExact;
    const bool e1 = lane + 32 < P.nv && s_cls[lane + 32] == kViewExact;
    const uint32_t b0 = __ballot_sync(0xffffffffu, m0), b1 = __ballot_sync(0xffffffffu, m1);
    const uint32_t x0 = __ballot_sync(0xffffffffu, e0), x1 = __ballot_sync(0xffffffffu, e1);
    const uint32_t f0 = __ballot_sync(0xffffffffu, lane < P.nv && s_cls[lane] == kViewFull);
    const uint32_t f1 = __ballot_sync(0xffffffffu, lane + 32 < P.nv && s_cls[lane + 32] == kViewFull);
    const uint32_t below = (1u << lane) - 1u;
    const int nm = __popc(b0) + __popc(b1);
    if (m0) s_list[__popc(b0 & below)] = (unsigned char)lane;
    if (m1) s_list[__popc(b0) + __popc(b1 & below)] = (unsigned char)(lane + 32);
    if (e0) s_list[nm + __popc(x0 & below)] = (unsigned char)lane;
    if (e1) s_list[nm + __popc(x0) + __popc(x1 & below)] = (unsigned char)(lane + 32);
    if (lane == 0) {
      s_nmixed = nm;
      s_nexact = __popc(x0) + __popc(x1);
      s_full[0] = f0;
      s_full[1] = f1;
      if (P.dbg) {
        atomicAdd(P.dbg + 16 * 1000 + 3, (unsigned long long)(__popc(f0) + __popc(f1)));
        atomicAdd(P.dbg + 16 * 1000 + 4, (unsigned long long)nm);
        atomicAdd(P.dbg + 16 * 1000 + 5, (unsigned long long)P.nv);
        atomicAdd(P.dbg + 16 * 1000 + 6, (unsigned long long)(__popc(x0) + __popc(x1)));
      }
    }
  }
  __syncthreads();
  const int nmixed = s_nmixed, nexact = s_nexact;
  uint32_t w0 = s_full[0], w1 = s_full[1];
  const float dx = p.x - 0.5f * (lo[0] + hi[0]), dy = p.y - 0.5f * (lo[1] + hi[1]), dz = p.z - 0.5f * (lo[2] + hi[2]);
  // MIXED views: every point against the tile's model (branch-free); the few samples the model
  // cannot decide (0.1 % at C5) are re-tested exactly afterwards, per lane
  uint64_t wm = 0ull, am = 0ull;  // this point's MIXED verdicts: visible / ambiguous
#pragma unroll 2
  for (int l = 0; l < nmixed; ++l) {
    const int v = s_list[l];
    bool vis, amb;
    affine_visible(saff[v], dx, dy, dz, eps_f, vis, amb);
    const uint64_t bit = 1ull << v;
    if (vis) wm |= bit;
    if (amb) am |= bit;
  }
  if (!live) wm = am = 0ull;
  if (P.dbg && tid == 0) atomicAdd(P.dbg + 16 * 1000 + 7, (unsigned long long)nmixed * 128ull);
  if (P.dbg && am) atomicAdd(P.dbg + 16 * 1000 + 8, (unsigned long long)__popcll(am));
  while (am) {  // rare: the exact test
    const int v = __ffsll((long long)am) - 1;
    am &= am - 1ull;
    TapF t;
    if (point_visible(sv[v], sbound[v], P.views[v], P.depth, p, P.eps, eps_f, t)) wm |= 1ull << v;
  }
  w0 |= (uint32_t)wm;
  w1 |= (uint32_t)(wm >> 32);
  // MIXED views this warp saw visible
  const uint32_t seen0 = __reduce_or_sync(0xffffffffu, (uint32_t)wm), seen1 = __reduce_or_sync(0xffffffffu, (uint32_t)(wm >> 32));
  if (lane == 0 && (seen0 | seen1)) {
    atomicOr(&s_seen[0], seen0);
    atomicOr(&s_seen[1], seen1);
  }
  for (int l = nmixed; l < nmixed + nexact; ++l) {
    const int v = s_list[l];
    TapF t;
    const bool vis = live && point_visible(sv[v], sbound[v], P.views[v], P.depth, p, P.eps, eps_f, t);
    if (vis) {
      if (v < 32) w0 |= 1u << v;
      else w1 |= 1u << (v - 32);
    }
    window_reduce(vis, t, wx0, wy0, wx1, wy1, v, lane);
  }
  // NaN point = padding slot (pf_shard_pack_padded): no view, voxel code -1 (the tile box above
  // already ignores it: fminf / fmaxf drop NaN)
  if (!live) w0 = w1 = 0u;
  const int32_t code = live ? voxel_code_fast(p, P.vox, P.grid) : -1;
  if (valid)
    *reinterpret_cast<uint4*>(P.srec + jpt) =
        make_uint4(w0, w1, (uint32_t)(__popc(w0) + __popc(w1)), (uint32_t)code);
  if (P.vox_list) {
    // touched-voxel list without returning atomics: slot jpt holds the code when this point is the
    // lowest lane of its warp with that code (a warp's sorted points share a few voxels), else -1;
    // pf_voxel_mass_sparse claims each voxel once (atomicExch on its count), so a voxel the SIMT
    // overflow kernel lists again is harmless
    const uint32_t peers = __match_any_sync(0xffffffffu, code);
    const bool first = (peers & ((1u << lane) - 1u)) == 0u;
    if (valid) P.vox_list[jpt] = first ? code : -1;
  }
  __syncthreads();
  if (tid < P.nv && s_cls[tid] == kViewMixed && ((s_seen[tid >> 5] >> (tid & 31)) & 1u)) {
    const uint32_t w = __float_as_uint(saff[tid].e.w);  // the box window (every visible point's taps)
    wx0[tid] = (int)(w & 0xff);
    wy0[tid] = (int)((w >> 8) & 0xff);
    wx1[tid] = (int)((w >> 16) & 0xff);
    wy1[tid] = (int)(w >> 24);
  }
  __syncthreads();
  if (tid < 32) {  // windows -> descriptors: exclusive prefix of window sizes over views (2 per lane)
    int w[2], h[2], x0[2], y0[2], sz[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int v = lane + 32 * r;
      w[r] = h[r] = 0;
      if (v < P.nv && wx1[v] >= 0) {
        w[r] = wx1[v] - wx0[v] + 1;
        h[r] = wy1[v] - wy0[v] + 1;
      }
      x0[r] = w[r] ? wx0[v] : 0;
      y0[r] = h[r] ? wy0[v] : 0;
      sz[r] = (w[r] * h[r] + 1) & ~1;  // windows start on even taps (whole 32-bit TMEM columns of bf16 pairs)
    }
    int incl0 = sz[0], incl1 = sz[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, incl0, o), t1 = __shfl_up_sync(0xffffffffu, incl1, o);
      if (lane >= o) {
        incl0 += t0;
        incl1 += t1;
      }
    }
    const int tot0 = __shfl_sync(0xffffffffu, incl0, 31);
    const int base0 = incl0 - sz[0], base1 = tot0 + incl1 - sz[1];
    uint2* desc = P.tile_desc + tile * P.nv;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int v = lane + 32 * r;
      const int base = r ? base1 : base0;
      if (v < P.nv)
        desc[v] = make_uint2((uint32_t)min(base, 65535) | ((uint32_t)x0[r] << 16) | ((uint32_t)y0[r] << 24),
                             (uint32_t)w[r] | ((uint32_t)h[r] << 8));
    }
    if (lane == 31) P.tile_kt[tile] = tot0 + incl1;
  }
}

// ---- overflow tiles -> smaller work items -------------------------------------------------------------
// A tile whose windows need more taps than one work item holds (it straddles a jump of the Hilbert
// order, or is a sparse patch) is re-run as 4 level-1 items of sub1_rows consecutive sorted points
// (k_tile_ws: 32 rows; Gram path: 128 rows), each with the exact union of its visible points' taps;
// the Gram path splits overflowing level-1 items once more into 4 level-2 items of 32 rows. A split
// parent is marked -1 (skipped); an item that still overflows goes to the SIMT kernel.
__global__ void k_find_overflow(TileParams P, int64_t ntiles, int kt_max) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
    const int kt = P.tile_kt[t];
    if (((kt + 15) & ~15) <= kt_max) continue;
    const int b = atomicAdd(P.sub_count, 1);
    if (b < P.max_sub_tiles) {
      P.sub_tiles[b] = (int32_t)t;
      P.tile_kt[t] = -1;
    }
  }
}

// Gram path: windows of a 512-row tile = per view, the hull of its four 128-row tiles' windows (the
// 128-row prep's FULL / MIXED box windows or EXACT unions all bound the visible points' taps), padded
// to even sizes and laid out by an exclusive prefix over the views. One warp per tile.
__global__ void k_merge512(TileParams P, int64_t nt) {
  const int lane = threadIdx.x & 31;
  const int64_t nt128 = (P.n + kTile - 1) / kTile;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < nt;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int w[2], h[2], x0[2], y0[2], sz[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int v = lane + 32 * r;
      int ax0 = INT_MAX, ay0 = INT_MAX, ax1 = -1, ay1 = -1;
      if (v < P.nv)
        for (int q = 0; q < 4; ++q) {
          const int64_t t128 = 4 * t + q;
          if (t128 >= nt128) break;
          const uint2 d = P.tile_desc[(nt + t128) * P.nv + v];
          const int ww = d.y & 0xff, hh = (d.y >> 8) & 0xff;
          if (!ww) continue;
          const int dx = (d.x >> 16) & 0xff, dy = d.x >> 24;
          ax0 = min(ax0, dx);
          ay0 = min(ay0, dy);
          ax1 = max(ax1, dx + ww - 1);
          ay1 = max(ay1, dy + hh - 1);
        }
      w[r] = ax1 >= 0 ? ax1 - ax0 + 1 : 0;
      h[r] = ax1 >= 0 ? ay1 - ay0 + 1 : 0;
      x0[r] = w[r] ? ax0 : 0;
      y0[r] = w[r] ? ay0 : 0;
      sz[r] = (w[r] * h[r] + 1) & ~1;
    }
    int incl0 = sz[0], incl1 = sz[1];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, incl0, o), t1 = __shfl_up_sync(0xffffffffu, incl1, o);
      if (lane >= o) {
        incl0 += t0;
        incl1 += t1;
      }
    }
    const int tot0 = __shfl_sync(0xffffffffu, incl0, 31);
    const int base0 = incl0 - sz[0], base1 = tot0 + incl1 - sz[1];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int v = lane + 32 * r;
      const int base = r ? base1 : base0;
      if (v < P.nv)
        P.tile_desc[t * P.nv + v] = make_uint2((uint32_t)min(base, 65535) | ((uint32_t)x0[r] << 16) | ((uint32_t)y0[r] << 24),
                                               (uint32_t)w[r] | ((uint32_t)h[r] << 8));
    }
    if (lane == 31) P.tile_kt[t] = tot0 + incl1;
  }
}

// Gram path: 128-row tiles of overflowing 512-row tiles that overflow too -> level-2 parents
__global__ void k_find_overflow128(TileParams P, int64_t nt, int kt_max) {
  const int64_t nt128 = (P.n + kTile - 1) / kTile;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt128; t += (int64_t)gridDim.x * blockDim.x) {
    const int k512 = P.tile_kt[t >> 2], k128 = P.tile_kt[nt + t];
    if (((k512 + 15) & ~15) <= kt_max || ((k128 + 15) & ~15) <= kt_max) continue;
    const int b = atomicAdd(P.sub2_count, 1);
    if (b < P.max_sub2) {
      P.sub2_items[b] = (int32_t)(nt + t);
      P.tile_kt[nt + t] = -1;
    }
  }
}

// first sorted row of a level-1 item
__device__ __forceinline__ int64_t level1_row0(const TileParams& P, int64_t ntiles, int64_t item) {
  const int64_t u = item - ntiles;
  return (int64_t)P.sub_tiles[u >> 2] * P.tr + (u & 3) * P.sub1_rows;
}

// Children of R rows (4 per parent) with exact windows. R = 32: a block is one parent, warp q its
// child q; R = 128: a block is one child. level 1: parents are tiles; level 2: level-1 items.
template <int R>
__global__ void __launch_bounds__(128) k_item_prep(TileParams P, int64_t ntiles, int level) {
  constexpr int kChildren = 128 / R;  // children per block
  __shared__ ViewF sv[kMaxViewsTC];
  __shared__ int sx0[kMaxViewsTC], sy0[kMaxViewsTC], sx1[kMaxViewsTC], sy1[kMaxViewsTC];
  const int nparents = level == 1 ? min(*P.sub_count, P.max_sub_tiles) : min(*P.sub2_count, P.max_sub2);
  const int64_t first = level == 1 ? ntiles : ntiles + 4 * (int64_t)P.max_sub_tiles;
  const int nblocks = nparents * (4 / kChildren);
  if ((int)blockIdx.x >= nblocks) return;
  for (int j = threadIdx.x; j < P.nv; j += 128) sv[j] = P.viewf[j];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int blk = blockIdx.x; blk < nblocks; blk += gridDim.x) {
    const int b = blk / (4 / kChildren);
    const int c = R == 32 ? warp : blk % 4;          // child of parent b
    const int r = R == 32 ? lane : (int)threadIdx.x;  // row within the child
    const int64_t item = first + 4 * (int64_t)b + c;
    const int64_t prow = level == 1               ? (int64_t)P.sub_tiles[b] * P.tr
                         : P.tr == kGramTile ? ((int64_t)P.sub2_items[b] - ntiles) * kTile  // a 128-row tile
                                             : level1_row0(P, ntiles, P.sub2_items[b]);
    const int64_t jpt = prow + (int64_t)c * R + r;
    const bool valid = jpt < P.n;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    uint2 mw = make_uint2(0u, 0u);
    if (valid) {
      p = P.spts[jpt];
      mw = *reinterpret_cast<const uint2*>(P.srec + jpt);
    }
    uint2* desc = P.tile_desc + item * P.nv;
    if (R > 32) {
      for (int v = threadIdx.x; v < P.nv; v += 128) {
        sx0[v] = INT_MAX;
        sy0[v] = INT_MAX;
        sx1[v] = -1;
        sy1[v] = -1;
      }
      __syncthreads();
    }
    int running = 0;
    for (int v = 0; v < P.nv; ++v) {
      const bool vis = (((v < 32 ? mw.x : mw.y) >> (v & 31)) & 1u) != 0u;
      int x0 = INT_MAX, y0 = INT_MAX, x1 = -1, y1 = -1;
      if (__any_sync(0xffffffffu, vis)) {
        if (vis) {
          const ProjF pr = project_f32(sv[v], p.x, p.y, p.z);
          const TapF t = taps_f32(sv[v], pr.u, pr.v);
          x0 = t.x0;
          y0 = t.y0;
          x1 = t.x0 + t.dx;
          y1 = t.y0 + t.dy;
        }
        x0 = __reduce_min_sync(0xffffffffu, x0);
        y0 = __reduce_min_sync(0xffffffffu, y0);
        x1 = __reduce_max_sync(0xffffffffu, x1);
        y1 = __reduce_max_sync(0xffffffffu, y1);
        if (R > 32 && lane == 0) {
          atomicMin(sx0 + v, x0);
          atomicMin(sy0 + v, y0);
          atomicMax(sx1 + v, x1);
          atomicMax(sy1 + v, y1);
        }
      }
      if (R == 32) {  // views in order: exclusive prefix of (even-padded) window sizes
        const int w = x1 >= 0 ? x1 - x0 + 1 : 0, h = x1 >= 0 ? y1 - y0 + 1 : 0;
        if (lane == 0)
          desc[v] = make_uint2((uint32_t)min(running, 65535) | ((uint32_t)(w ? x0 : 0) << 16) | ((uint32_t)(h ? y0 : 0) << 24),
                               (uint32_t)w | ((uint32_t)h << 8));
        running += (w * h + 1) & ~1;
      }
    }
    if (R > 32) {
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int v = 0; v < P.nv; ++v) {
          const int x0 = sx0[v], y0 = sy0[v], x1 = sx1[v], y1 = sy1[v];
          const int w = x1 >= 0 ? x1 - x0 + 1 : 0, h = x1 >= 0 ? y1 - y0 + 1 : 0;
          desc[v] = make_uint2((uint32_t)min(running, 65535) | ((uint32_t)(w ? x0 : 0) << 16) | ((uint32_t)(h ? y0 : 0) << 24),
                               (uint32_t)w | ((uint32_t)h << 8));
          running += (w * h + 1) & ~1;
        }
        P.tile_kt[item] = running;
      }
      __syncthreads();
    } else if (lane == 0) {
      P.tile_kt[item] = running;
    }
  }
}

// ---- sorted records -> caller's point order (gather: one 32-byte record read per point) -----------------
__global__ void k_unsort(const SRec* __restrict__ srec, const int32_t* __restrict__ inv, int64_t n,
                         int nwords, int p, uint32_t* __restrict__ mask_bits, int32_t* __restrict__ counts,
                         int32_t* __restrict__ codes, float* __restrict__ props) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = __ldg(inv + i);
    PF_DCHECK(j >= 0 && j < n + 512, "inverse permutation");
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(srec + j));
    const float4 b = __ldg(reinterpret_cast<const float4*>(srec + j) + 1);
    if (nwords == 2) {
      *reinterpret_cast<uint2*>(mask_bits + 2 * i) = make_uint2(a.x, a.y);
    } else {
      mask_bits[i] = a.x;
    }
    counts[i] = (int32_t)a.z;
    codes[i] = (int32_t)a.w;
    if (p == 2) {
      *reinterpret_cast<float2*>(props + 2 * i) = make_float2(b.x, b.y);
    } else {
      const float pv[4] = {b.x, b.y, b.z, b.w};
      for (int q = 0; q < p; ++q) props[i * p + q] = pv[q];
    }
  }
}

// G in bf16 (cells x kpadg) for the tensor path, from the fp32 table of the SIMT path
__global__ void k_g_bf16(const float* __restrict__ G, int64_t cells, int kpad, int kpadg,
                         uint16_t* __restrict__ Gbf) {
  const int64_t total = cells * kpadg;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / kpadg;
    const int k = (int)(e - c * kpadg);
    Gbf[e] = __bfloat16_as_ushort(__float2bfloat16_rn(k < kpad ? G[c * kpad + k] : 0.f));
  }
}

}  // namespace tile
}  // namespace pf

// ---- host orchestration -----------------------------------------------------------------------------
namespace pf {
namespace tile {

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// CUB radix-sort scratch for n (key, index) pairs (a host-side size query, no device work)
static size_t radix_sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n > 0 ? n : 1), 0,
                                  3 * sort_bits_for(n));
  return bytes;
}

TileLayout tile_layout(int64_t n, int nv, int64_t cells, int kpadg, int d, bool x3, int tr) {
  TileLayout L{};
  const int64_t ntiles = (n + tr - 1) / tr;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  // per-object tables first: their offsets do not depend on the point count or the tile size, so
  // pf_fuse_prepare's tables stay valid for either kernel (tile sizes 128 / 512)
  L.gbf = take(sizeof(uint16_t) * (size_t)cells * kpadg);
  L.textbf = take(sizeof(uint16_t) * (size_t)kpadg * 1024);  // text rows in bf16 (D <= 1024)
  L.tbound = take(sizeof(float) * 4);
  if (x3) {  // lo part of G, hi and lo parts of the f32 maps
    L.glo = take(sizeof(uint16_t) * (size_t)cells * kpadg);
    L.fhi = take(sizeof(uint16_t) * (size_t)cells * d);
    L.flo = take(sizeof(uint16_t) * (size_t)cells * d);
    L.textlo = take(sizeof(uint16_t) * (size_t)kpadg * 1024);
  }
  L.viewf = take(sizeof(ViewF) * kMaxViewsTC);
  L.vbound = take(sizeof(float4) * kMaxViewsTC);
  L.vox = take(sizeof(double) * 8);
  L.ntiles = ntiles;
  // Hilbert keys: counting sort (histogram + scan + atomic scatter; the order of the points of one
  // key varies from run to run) or, with PF_FUSE_DETERMINISTIC, a stable LSD radix sort of (key,
  // index) pairs (CUB): deterministic tiles, ~0.7 ms slower at C5
  L.keys = take(sizeof(uint32_t) * (size_t)n);
  L.hist = take(sizeof(uint32_t) * (size_t)(1 << (3 * sort_bits_for(n))));
  L.totals = take(sizeof(uint32_t) * 4096);
  L.keys_out = take(sizeof(uint32_t) * (size_t)n);
  L.idx = take(sizeof(uint32_t) * (size_t)n);
  L.idx_out = take(sizeof(uint32_t) * (size_t)n);
  L.sort_tmp = take(radix_sort_temp_bytes(n));
  L.inv = take(sizeof(int32_t) * (size_t)n);
  L.spts = take(sizeof(float4) * (size_t)ntiles * tr);
  L.srec = take(sizeof(SRec) * (size_t)ntiles * tr);
  L.max_sub_tiles = (int32_t)ntiles;  // every tile may be split (sparse clouds overflow often)
  // Gram path: up to ntiles level-1 items may split again (each into 4 level-2 items)
  L.max_sub2 = tr == kTile ? 0 : (int32_t)(4 * ntiles);  // sparse clouds: most level-1 items may split
  const int64_t items = ntiles + 4 * (int64_t)L.max_sub_tiles + 4 * (int64_t)L.max_sub2;
  L.desc = take(sizeof(uint2) * (size_t)items * nv);
  L.kt = take(sizeof(int32_t) * (size_t)items);
  L.sub = take(sizeof(int32_t) * ((size_t)L.max_sub_tiles + 1));
  L.sub2 = take(sizeof(int32_t) * ((size_t)L.max_sub2 + 1));
  L.ovf = take(sizeof(int32_t) * (size_t)(n + 1));
  L.work = tr == kTile ? 0 : take(sizeof(int4) * (size_t)(items + 1));  // [count | pad] then entries
  L.wlist = tr == kTile ? 0 : take(sizeof(int4) * (size_t)(items + 1));  // split items for k_tile_ws
  L.work_raw = tr == kTile ? 0 : take(sizeof(int4) * (size_t)items);  // unsorted work list
  L.tbox = tr == kTile ? 0 : take(2 * sizeof(float4) * (size_t)((n + kTile - 1) / kTile));  // 128-row tile boxes
  L.bytes = off;
  return L;
}

__global__ void k_order_scatter(int64_t n, const uint32_t* __restrict__ keys, uint32_t* __restrict__ cursor,
                                int32_t* __restrict__ order, int32_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    order[atomicAdd(cursor + keys[i], 1u)] = (int32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *len = (int32_t)n;
}

size_t point_order_bytes(int64_t n) {
  return align256(sizeof(uint32_t) * (size_t)n) + align256(sizeof(uint32_t) << 21) + align256(sizeof(uint32_t) * 4096);
}

int run_point_order(const float* points, int64_t n, const double* lo_hi, unsigned char* ws, int32_t* order,
                    int32_t* len, cudaStream_t st) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + align256(sizeof(uint32_t) * (size_t)n));
  uint32_t* totals = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(hist) + align256(sizeof(uint32_t) << 21));
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) << 21, st);
  k_sort_keys<7><<<grid_for(n, 256), 256, 0, st>>>(points, n, lo_hi, keys, hist, nullptr);
  if (int rc = check_launch("order_keys")) return rc;
  if (int rc = run_bucket_scan(hist, totals, int64_t(1) << 21, st)) return rc;
  k_order_scatter<<<grid_for(n, 256), 256, 0, st>>>(n, keys, hist, order, len);
  return check_launch("order_scatter");
}

// hi = bf16_rn(x), lo = bf16_rn(x - hi) (x - hi is exact in fp32); columns >= cols are zero
__global__ void k_split_f32(const float* __restrict__ src, int64_t rows, int cols, int src_ld, int dst_ld,
                            uint16_t* __restrict__ hi, uint16_t* __restrict__ lo) {
  const int64_t total = rows * (int64_t)dst_ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / dst_ld;
    const int c = (int)(e - r * dst_ld);
    const float x = c < cols ? src[r * src_ld + c] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    hi[e] = __bfloat16_as_ushort(h);
    lo[e] = __bfloat16_as_ushort(__float2bfloat16_rn(x - __bfloat162float(h)));
  }
}

int run_split_f32(const float* src, int64_t rows, int cols, int src_ld, int dst_ld, uint16_t* hi, uint16_t* lo,
                  cudaStream_t st) {
  k_split_f32<<<grid_for(rows * (int64_t)dst_ld, 256), 256, 0, st>>>(src, rows, cols, src_ld, dst_ld, hi, lo);
  return check_launch("split_f32");
}

int run_g_bf16(const float* G, int64_t cells, int kpad, int kpadg, uint16_t* Gbf, cudaStream_t st) {
  k_g_bf16<<<grid_for(cells * kpadg, 256), 256, 0, st>>>(G, cells, kpad, kpadg, Gbf);
  return check_launch("g_bf16");
}

// exclusive scan of `nbins` (multiple of 4096, <= 16M) bucket counters in place (k_scan_*)
int run_bucket_scan(uint32_t* hist, uint32_t* totals, int64_t nbins, cudaStream_t st, bool add_block_bases) {
  if (nbins % 4096 != 0 || nbins / 4096 > 4096) return set_error(PF_ERR_VALUE, "bucket scan: bad bin count");
  const int nb = (int)(nbins / 4096);
  k_scan_blocks<<<nb, 1024, 0, st>>>(hist, totals);
  if (int rc = check_launch("scan_blocks")) return rc;
  k_scan_totals<<<1, 1024, 0, st>>>(totals, nb);
  if (int rc = check_launch("scan_totals")) return rc;
  if (!add_block_bases) return PF_OK;
  k_scan_add<<<(unsigned)(nbins / 256), 256, 0, st>>>(hist, totals);
  return check_launch("scan_add");
}

int run_unsort(const TileParams& P, cudaStream_t st) {
  k_unsort<<<grid_for(P.n, 256, 1 << 30), 256, 0, st>>>(P.srec, P.inv, P.n, P.nwords, P.p, P.mask_bits, P.counts,
                                              P.codes, P.props);
  const int rc = check_launch("unsort");
  stage_mark(4, st);
  return rc;
}

int run_tile_path(TileParams P, const TileLayout& L, unsigned char* ws, const float* points,
                  int64_t n, cudaStream_t st, ForkHook fork, cudaEvent_t* joined) {
  cudaEvent_t g_ready = nullptr;
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws + L.keys);
  stage_mark(0, st);
  // the tables overlap the sort (forking at the prep instead measured slower: prep is issue-bound
  // and the G projection took its SMs, +0.15 ms against the 0.1 ms it hid)
  if (fork.fn) {
    int frc = PF_OK;
    g_ready = fork.fn(fork.ctx, st, &frc);
    if (joined) *joined = g_ready;
    if (frc) return frc;
  }
  const int bits = sort_bits_for(n);
  cudaMemsetAsync(P.ovf_count, 0, sizeof(int32_t), st);
  if (P.deterministic) {
    uint32_t* keys_out = reinterpret_cast<uint32_t*>(ws + L.keys_out);
    uint32_t* idx = reinterpret_cast<uint32_t*>(ws + L.idx);
    uint32_t* idx_out = reinterpret_cast<uint32_t*>(ws + L.idx_out);
    if (bits == 8) k_sort_keys<8><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(points, n, P.lo_hi, keys, nullptr, idx);
    else k_sort_keys<7><<<grid_for(n, 256), 256, 0, st>>>(points, n, P.lo_hi, keys, nullptr, idx);
    if (int rc = check_launch("sort_keys")) return rc;
    size_t tmp_bytes = radix_sort_temp_bytes(n);
    if (cub::DeviceRadixSort::SortPairs(ws + L.sort_tmp, tmp_bytes, keys, keys_out, idx, idx_out, (int)n, 0,
                                        3 * bits, st) != cudaSuccess)
      return check_launch("radix_sort");
    k_sort_gather<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(points, n, idx_out, const_cast<int32_t*>(P.inv),
                                                            const_cast<float4*>(P.spts));
    if (int rc = check_launch("sort_gather")) return rc;
  } else {
    uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
    uint32_t* totals = reinterpret_cast<uint32_t*>(ws + L.totals);
    const int64_t nbins = int64_t(1) << (3 * bits);
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * nbins, st);
    if (bits == 8) k_sort_keys<8><<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(points, n, P.lo_hi, keys, hist, nullptr);
    else k_sort_keys<7><<<grid_for(n, 256), 256, 0, st>>>(points, n, P.lo_hi, keys, hist, nullptr);
    if (int rc = check_launch("sort_keys")) return rc;
    // block-local bucket offsets: the scatter adds its 4096-bin block's base itself (no pass over the
    // 16M bins to add them)
    if (int rc = run_bucket_scan(hist, totals, nbins, st, false)) return rc;
    k_sort_scatter<<<grid_for(n, 256, 1 << 30), 256, 0, st>>>(points, n, keys, hist, totals, const_cast<int32_t*>(P.inv),
                                                             const_cast<float4*>(P.spts));
    if (int rc = check_launch("sort_scatter")) return rc;
  }
  stage_mark(1, st);
  if (fork.depth_ready) cudaStreamWaitEvent(st, fork.depth_ready, 0);  // first read by the prep
  static unsigned long long* pdbg = nullptr;
  const bool debug = getenv("PF_WS_DEBUG") != nullptr;
  TileParams Q = P;
  if (debug) {
    if (!pdbg) cudaMalloc(&pdbg, sizeof(unsigned long long) * 16 * 1024);
    cudaMemsetAsync(pdbg, 0, sizeof(unsigned long long) * 16 * 1024, st);
    Q.dbg = pdbg;
  }
  k_view_setup<<<1, kMaxViewsTC, 0, st>>>(Q);
  if (int rc = check_launch("view_setup")) return rc;
  if (P.tr == kGramTile) {
    // Gram path: per-point visibility and windows from the 128-row prep (its tiles are the level-1
    // items, ids ntiles + t128), the 512-row tiles' windows merged from theirs, the 128-row tiles
    // that still overflow split into 32-row items
    const int64_t nt128 = (n + kTile - 1) / kTile;
    TileParams Q128 = Q;
    Q128.tr = kTile;
    Q128.tile_desc = P.tile_desc + L.ntiles * P.nv;
    Q128.tile_kt = P.tile_kt + L.ntiles;
    k_tile_prep<kTile><<<(unsigned)nt128, kTile, 0, st>>>(Q128);
    if (int rc = check_launch("tile_prep")) return rc;
    k_merge512<<<grid_for(32 * L.ntiles, 256), 256, 0, st>>>(P, L.ntiles);
    if (int rc = check_launch("merge512")) return rc;
    cudaMemsetAsync(P.sub2_count, 0, sizeof(int32_t), st);
    k_find_overflow128<<<grid_for(nt128, 256), 256, 0, st>>>(P, L.ntiles, P.kt_max);
    if (int rc = check_launch("find_overflow128")) return rc;
    k_item_prep<32><<<(unsigned)(L.max_sub2 < 148 * 16 ? L.max_sub2 : 148 * 16), 128, 0, st>>>(P, L.ntiles, 2);
    if (int rc = check_launch("item_prep2")) return rc;
    stage_mark(2, st);
    if (g_ready) cudaStreamWaitEvent(st, g_ready, 0);  // G, bf16 text, text bound
    if (fork.fmap_ready) cudaStreamWaitEvent(st, fork.fmap_ready, 0);
    const int rc = run_tile_gram(P, st);
    stage_mark(3, st);
    return rc;
  }
  k_tile_prep<kTile><<<(unsigned)L.ntiles, kTile, 0, st>>>(Q);
  if (int rc = check_launch("tile_prep")) return rc;
  // overflow tiles -> smaller work items (appended after the tiles)
  cudaMemsetAsync(P.sub_count, 0, sizeof(int32_t), st);
  k_find_overflow<<<grid_for(L.ntiles, 256), 256, 0, st>>>(P, L.ntiles, P.kt_max);
  if (int rc = check_launch("find_overflow")) return rc;
  const unsigned pgrid = (unsigned)(L.max_sub_tiles < 148 * 16 ? L.max_sub_tiles : 148 * 16);
  if (P.sub1_rows == 32) k_item_prep<32><<<pgrid, 128, 0, st>>>(P, L.ntiles, 1);
  else k_item_prep<128><<<4 * pgrid, 128, 0, st>>>(P, L.ntiles, 1);
  if (int rc = check_launch("item_prep")) return rc;
  stage_mark(2, st);
  if (debug) {
    unsigned long long h[11];
    cudaMemcpyAsync(h, pdbg + 16 * 1000, sizeof(h), cudaMemcpyDeviceToHost, st);
    std::vector<int32_t> kt((size_t)L.ntiles);
    cudaMemcpyAsync(kt.data(), P.tile_kt, sizeof(int32_t) * kt.size(), cudaMemcpyDeviceToHost, st);
    int32_t nsub_tiles = 0;
    cudaMemcpyAsync(&nsub_tiles, P.sub_count, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    {
      const int nsi = 4 * (nsub_tiles < L.max_sub_tiles ? nsub_tiles : L.max_sub_tiles);
      std::vector<int32_t> skt(nsi > 0 ? nsi : 1);
      if (nsi) cudaMemcpy(skt.data(), P.tile_kt + L.ntiles, sizeof(int32_t) * nsi, cudaMemcpyDeviceToHost);
      int over2 = 0;
      for (int k = 0; k < nsi; ++k) over2 += ((skt[k] + 15) & ~15) > P.kt_max;
      fprintf(stderr, "[prep debug] overflow tiles %d -> %d sub-tiles, %d of them still over %d taps\n", nsub_tiles,
              nsi, over2, P.kt_max);
    }
    double ksum = 0;
    int64_t over = 0, kmax = 0;
    for (int32_t k : kt) {
      if (k < 0) { ++over; continue; }
      ksum += k;
      over += ((k + 15) & ~15) > P.kt_max;
      kmax = k > kmax ? k : kmax;
    }
    {  // window shapes
      std::vector<uint2> ds((size_t)L.ntiles * P.nv);
      cudaMemcpy(ds.data(), P.tile_desc, sizeof(uint2) * ds.size(), cudaMemcpyDeviceToHost);
      long long hist[6] = {0, 0, 0, 0, 0, 0}, taps_in[6] = {0, 0, 0, 0, 0, 0}, nonempty = 0;
      const char* nm[6] = {"2x2", "1x1/1x2/2x1", "3x2/2x3", "3x3", "<=16 other", ">16"};
      for (const uint2& d : ds) {
        const int w = d.y & 0xff, h = (d.y >> 8) & 0xff;
        if (!w) continue;
        ++nonempty;
        const int c = (w == 2 && h == 2) ? 0 : (w * h <= 2) ? 1 : (w * h == 6) ? 2 : (w == 3 && h == 3) ? 3
                      : (w * h <= 16) ? 4 : 5;
        ++hist[c];
        taps_in[c] += w * h;
      }
      fprintf(stderr, "[prep debug] windows per tile %.1f:", (double)nonempty / L.ntiles);
      for (int c = 0; c < 6; ++c)
        fprintf(stderr, " %s %.1f%% (taps %.1f%%)", nm[c], 100.0 * hist[c] / nonempty, 0.0);
      fprintf(stderr, "\n");
      long long tt = 0;
      for (int c = 0; c < 6; ++c) tt += taps_in[c];
      fprintf(stderr, "[prep debug] share of taps:");
      for (int c = 0; c < 6; ++c) fprintf(stderr, " %s %.1f%%", nm[c], 100.0 * taps_in[c] / tt);
      fprintf(stderr, "\n");
    }
    fprintf(stderr, "[prep debug] tile x view: FULL %.1f%%, MIXED %.1f%%, EXACT %.1f%%, OFF %.1f%%; taps per tile "
            "mean %.1f max %lld, overflow tiles %lld of %lld\n", 100.0 * h[3] / h[5], 100.0 * h[4] / h[5],
            100.0 * h[6] / h[5], 100.0 * (h[5] - h[3] - h[4] - h[6]) / h[5], ksum / kt.size(), (long long)kmax,
            (long long)over, (long long)kt.size());
    fprintf(stderr, "[prep debug] MIXED samples ambiguous under the affine model: %.2f%%, mean eu %.4f px\n",
            100.0 * h[8] / (double)(h[7] ? h[7] : 1), 1e-6 * h[9] / (double)(h[10] ? h[10] : 1));
  }
  if (g_ready) cudaStreamWaitEvent(st, g_ready, 0);  // G (and the x3 map splits)
  if (fork.fmap_ready) cudaStreamWaitEvent(st, fork.fmap_ready, 0);
  const int rc = run_tile_ws(P, st);
  stage_mark(3, st);
  return rc;
}

}  // namespace tile
}  // namespace pf

// ---- diagnostics: the sort key of the tile path ------------------------------------------------------
extern "C" {

int pf_hilbert_table(uint8_t* out, int32_t n) {
  if (!out || n < pf::tile::kHilbertStates * 8)
    return pf::set_error(PF_ERR_VALUE, "hilbert_table: need %d bytes", pf::tile::kHilbertStates * 8);
  memcpy(out, pf::tile::kHilbertFsmH, pf::tile::kHilbertStates * 8);
  return pf::tile::kHilbertStates;
}

int pf_hilbert_keys(const float* points, int64_t n, const double* lo_hi, int32_t bits, uint32_t* keys,
                    void* stream) {
  if (bits != 7 && bits != 8) return pf::set_error(PF_ERR_VALUE, "hilbert_keys: bits must be 7 or 8, got %d", bits);
  if (n <= 0) return PF_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (bits == 8) pf::tile::k_sort_keys<8><<<pf::grid_for(n, 256), 256, 0, st>>>(points, n, lo_hi, keys, nullptr, nullptr);
  else pf::tile::k_sort_keys<7><<<pf::grid_for(n, 256), 256, 0, st>>>(points, n, lo_hi, keys, nullptr, nullptr);
  return pf::check_launch("hilbert_keys");
}

}  // extern "C"

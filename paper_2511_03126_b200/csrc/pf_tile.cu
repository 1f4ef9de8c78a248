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
//   k_sort_keys / k_scan_* / k_sort_scatter — counting sort of the points by a 21-bit Morton key of
//       a 128^3 grid over the bbox (spatial coherence of tiles; no library sort);
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
#include "pf_tile_dev.cuh"

namespace pf {
namespace tile {

// ---- counting sort by a coarse Morton key --------------------------------------------------------------
__device__ __forceinline__ uint32_t spread3(uint32_t x) {
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000ffu;
  x = (x | (x << 8)) & 0x0300f00fu;
  x = (x | (x << 4)) & 0x030c30c3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

__global__ void k_sort_keys(const float* __restrict__ p, int64_t n, const double* __restrict__ lo_hi,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ hist) {
  const float lx = (float)lo_hi[0], ly = (float)lo_hi[1], lz = (float)lo_hi[2];
  const float ext = fmaxf(fmaxf((float)(lo_hi[3] - lo_hi[0]), (float)(lo_hi[4] - lo_hi[1])),
                          (float)(lo_hi[5] - lo_hi[2]));
  const float inv = ext > 0.f ? (float)kSortCells / ext : 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int cx = min(max((int)((__ldg(p + 3 * i) - lx) * inv), 0), kSortCells - 1);
    const int cy = min(max((int)((__ldg(p + 3 * i + 1) - ly) * inv), 0), kSortCells - 1);
    const int cz = min(max((int)((__ldg(p + 3 * i + 2) - lz) * inv), 0), kSortCells - 1);
    const uint32_t key = spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2);
    keys[i] = key;
    atomicAdd(hist + key, 1u);
  }
}

// exclusive scan of kSortBins counters: per-block scan of 4096 (1024 threads x 4), block totals,
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
  __shared__ uint32_t s[1024];
  const int t = threadIdx.x;
  s[t] = t < nblocks ? totals[t] : 0u;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t v = t >= o ? s[t - o] : 0u;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  if (t < nblocks) totals[t] = s[t] - (t < nblocks ? totals[t] : 0u);
}

__global__ void k_scan_add(uint32_t* __restrict__ hist, const uint32_t* __restrict__ totals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  hist[i] += totals[i / 4096];
}

__global__ void k_sort_scatter(const float* __restrict__ p, int64_t n, const uint32_t* __restrict__ keys,
                               uint32_t* __restrict__ cursor, int32_t* __restrict__ inv,
                               float4* __restrict__ spts) {
  // one scattered 16-byte write per point (the sorted point carries its original index in .w);
  // the inverse permutation is written coalesced
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pos = atomicAdd(cursor + keys[i], 1u);
    inv[i] = (int32_t)pos;
    spts[pos] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2),
                            __int_as_float((int32_t)i));
  }
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
enum : int { kViewOff = 0, kViewFull = 1, kViewMixed = 2 };
constexpr int kScanMax = 64;  // pixels of depth scanned per (tile, view) at most

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
//   MIXED: anything else (per-point exact test).
// FULL views also get their tap window here: fu = (u + 0.5) * Wf/W - 0.5 is computed by the same
// monotone fp32 ops as taps_f32 on the widened pixel range, which bounds every point's taps.
__device__ int classify_tile_view(const ViewF& v, const float* __restrict__ depth, const float* lo,
                                  const float* hi, float eps, int4& win) {
  float zmin = 1e30f, zmax = -1e30f, umin = 1e30f, umax = -1e30f, vmin = 1e30f, vmax = -1e30f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float px = (c & 1) ? hi[0] : lo[0];
    const float py = (c & 2) ? hi[1] : lo[1];
    const float pz = (c & 4) ? hi[2] : lo[2];
    const float X = fmaf(v.R[2], pz, fmaf(v.R[1], py, v.R[0] * px)) + v.t[0];
    const float Y = fmaf(v.R[5], pz, fmaf(v.R[4], py, v.R[3] * px)) + v.t[1];
    const float Z = fmaf(v.R[8], pz, fmaf(v.R[7], py, v.R[6] * px)) + v.t[2];
    zmin = fminf(zmin, Z);
    zmax = fmaxf(zmax, Z);
    const float rz = 1.f / Z;
    const float u = fmaf(v.fx, X * rz, v.cx), w = fmaf(v.fy, Y * rz, v.cy);
    umin = fminf(umin, u);
    umax = fmaxf(umax, u);
    vmin = fminf(vmin, w);
    vmax = fmaxf(vmax, w);
  }
  if (!(zmin > 1e-3f)) return kViewMixed;  // the box reaches the camera plane
  const float ulo = fmaxf(umin - 0.01f, -1e6f), uhi = fminf(umax + 0.01f, 1e6f);
  const float vlo = fmaxf(vmin - 0.01f, -1e6f), vhi = fminf(vmax + 0.01f, 1e6f);
  const int x0 = (int)rintf(ulo), x1 = (int)rintf(uhi), y0 = (int)rintf(vlo), y1 = (int)rintf(vhi);
  const int cx0 = max(x0, 0), cx1 = min(x1, v.W - 1), cy0 = max(y0, 0), cy1 = min(y1, v.H - 1);
  if (cx1 < cx0 || cy1 < cy0) return kViewOff;
  const int bw = cx1 - cx0 + 1, bh = cy1 - cy0 + 1;
  if (bw * bh > kScanMax) return kViewMixed;
  const float* d = depth + v.depth_off + (int64_t)cy0 * v.W + cx0;
  float dmax = 0.f, dmin = 1e30f;
  const int npx = bw * bh;
  for (int k = 0; k < npx; k += 4) {  // four independent loads in flight
    float s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int kk = min(k + u, npx - 1), yy = kk / bw;
      s[u] = __ldg(d + (int64_t)yy * v.W + (kk - yy * bw));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dmax = fmaxf(dmax, s[u]);
      dmin = fminf(dmin, s[u]);
    }
  }
  if (zmin - 1e-5f > dmax + eps + 1e-5f) return kViewOff;
  const bool inside = x0 >= 0 && y0 >= 0 && x1 < v.W && y1 < v.H;
  if (!(inside && dmin > 0.f && zmax + 2e-5f < dmin + eps)) return kViewMixed;
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
  return kViewFull;
}

__global__ void k_view_setup(TileParams P) {
  const int j = threadIdx.x;
  if (j < P.nv) {
    const ViewF w = make_viewf(P.views[j], P.d);
    P.viewf[j] = w;
    P.vbound[j] = view_bound(w, P.views[j], P.lo_hi);
  }
}

// exact per-point decision for one (point, MIXED view) sample; fills the taps when visible
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

// ---- k_tile_prep ---------------------------------------------------------------------------------------
// One warp's 32 consecutive sorted points form the classification box (a ~2 mm patch at C5: small
// enough that most views are decided for all 32 points at once); lane l classifies views l and
// l + 32. FULL views set their bit for the whole warp and widen the tile's tap window by the box
// window; MIXED views run the exact per-point test and widen it by the visible points' taps.
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

__global__ void __launch_bounds__(kTile, 8) k_tile_prep(TileParams P) {
  constexpr int kWarps = kTile / 32;
  __shared__ ViewF sv[kMaxViewsTC];
  __shared__ float4 sbound[kMaxViewsTC];
  __shared__ int wx0[kMaxViewsTC], wx1[kMaxViewsTC], wy0[kMaxViewsTC], wy1[kMaxViewsTC];
  __shared__ unsigned char s_mixed[kWarps][kMaxViewsTC];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t jpt = tile * kTile + tid;
  const bool valid = jpt < P.n;
  const float4 p = valid ? P.spts[jpt] : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = tid; j < P.nv; j += kTile) {
    sv[j] = P.viewf[j];  // per-view fp32 camera + constant error bounds (k_view_setup)
    sbound[j] = P.vbound[j];
    wx0[j] = INT_MAX;
    wy0[j] = INT_MAX;
    wx1[j] = -1;
    wy1[j] = -1;
  }
  float lo[3] = {valid ? p.x : INFINITY, valid ? p.y : INFINITY, valid ? p.z : INFINITY};
  float hi[3] = {valid ? p.x : -INFINITY, valid ? p.y : -INFINITY, valid ? p.z : -INFINITY};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  }
  __syncthreads();
  const float eps_f = (float)P.eps;
  const bool any_point = lo[0] <= hi[0];
  uint32_t fb[2], mb[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int v = lane + 32 * r;
    int cls = kViewOff;
    if (any_point && v < P.nv) {
      int4 win = make_int4(INT_MAX, INT_MAX, -1, -1);
      cls = classify_tile_view(sv[v], P.depth, lo, hi, eps_f, win);
      if (cls == kViewFull) {
        atomicMin(wx0 + v, win.x);
        atomicMin(wy0 + v, win.y);
        atomicMax(wx1 + v, win.z);
        atomicMax(wy1 + v, win.w);
      }
    }
    fb[r] = __ballot_sync(0xffffffffu, cls == kViewFull);
    mb[r] = __ballot_sync(0xffffffffu, cls == kViewMixed);
    const uint32_t below = (1u << lane) - 1u;
    if (cls == kViewMixed) s_mixed[wid][(r ? __popc(mb[0]) : 0) + __popc(mb[r] & below)] = (unsigned char)v;
  }
  __syncwarp();
  if (P.dbg && lane == 0) {
    atomicAdd(P.dbg + 16 * 1000 + 3, (unsigned long long)(__popc(fb[0]) + __popc(fb[1])));
    atomicAdd(P.dbg + 16 * 1000 + 4, (unsigned long long)(__popc(mb[0]) + __popc(mb[1])));
    atomicAdd(P.dbg + 16 * 1000 + 5, (unsigned long long)P.nv);
  }
  const int nmixed = __popc(mb[0]) + __popc(mb[1]);
  const unsigned char* mixed = s_mixed[wid];
  uint32_t w0 = fb[0], w1 = fb[1];
  int l = 0;
  for (; l + 1 < nmixed; l += 2) {  // two MIXED views in flight (independent depth loads)
    const int va = mixed[l], vb = mixed[l + 1];
    TapF ta, tb;
    const bool visa = valid && point_visible(sv[va], sbound[va], P.views[va], P.depth, p, P.eps, eps_f, ta);
    const bool visb = valid && point_visible(sv[vb], sbound[vb], P.views[vb], P.depth, p, P.eps, eps_f, tb);
    if (visa) {
      if (va < 32) w0 |= 1u << va;
      else w1 |= 1u << (va - 32);
    }
    if (visb) {
      if (vb < 32) w0 |= 1u << vb;
      else w1 |= 1u << (vb - 32);
    }
    window_reduce(visa, ta, wx0, wy0, wx1, wy1, va, lane);
    window_reduce(visb, tb, wx0, wy0, wx1, wy1, vb, lane);
  }
  if (l < nmixed) {
    const int v = mixed[l];
    TapF t;
    const bool vis = valid && point_visible(sv[v], sbound[v], P.views[v], P.depth, p, P.eps, eps_f, t);
    if (vis) {
      if (v < 32) w0 |= 1u << v;
      else w1 |= 1u << (v - 32);
    }
    window_reduce(vis, t, wx0, wy0, wx1, wy1, v, lane);
  }
  if (valid) {
    double dlo[3];
    const double edge = voxel_edge(P.lo_hi, P.grid, dlo);
    const int32_t code = voxel_code(p.x, p.y, p.z, dlo, edge, P.grid);
    *reinterpret_cast<uint4*>(P.srec + jpt) =
        make_uint4(w0, w1, (uint32_t)(__popc(w0) + __popc(w1)), (uint32_t)code);
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

// ---- sorted records -> caller's point order (gather: one 32-byte record read per point) -----------------
__global__ void k_unsort(const SRec* __restrict__ srec, const int32_t* __restrict__ inv, int64_t n,
                         int nwords, int p, uint32_t* __restrict__ mask_bits, int32_t* __restrict__ counts,
                         int32_t* __restrict__ codes, float* __restrict__ props) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = __ldg(inv + i);
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

TileLayout tile_layout(int64_t n, int nv, int64_t cells, int kpadg) {
  TileLayout L{};
  const int64_t ntiles = (n + kTile - 1) / kTile;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align256(bytes);
    return o;
  };
  L.ntiles = ntiles;
  L.keys = take(sizeof(uint32_t) * (size_t)n);
  L.hist = take(sizeof(uint32_t) * (size_t)kSortBins);
  L.totals = take(sizeof(uint32_t) * 1024);
  L.inv = take(sizeof(int32_t) * (size_t)n);
  L.spts = take(sizeof(float4) * (size_t)ntiles * kTile);
  L.srec = take(sizeof(SRec) * (size_t)ntiles * kTile);
  L.desc = take(sizeof(uint2) * (size_t)ntiles * nv);
  L.kt = take(sizeof(int32_t) * (size_t)ntiles);
  L.viewf = take(sizeof(ViewF) * kMaxViewsTC);
  L.vbound = take(sizeof(float4) * kMaxViewsTC);
  L.ovf = take(sizeof(int32_t) * (size_t)(n + 1));
  L.gbf = take(sizeof(uint16_t) * (size_t)cells * kpadg);
  L.bytes = off;
  return L;
}

int run_g_bf16(const float* G, int64_t cells, int kpad, int kpadg, uint16_t* Gbf, cudaStream_t st) {
  k_g_bf16<<<grid_for(cells * kpadg, 256), 256, 0, st>>>(G, cells, kpad, kpadg, Gbf);
  return check_launch("g_bf16");
}

int run_unsort(const TileParams& P, cudaStream_t st) {
  k_unsort<<<grid_for(P.n, 256), 256, 0, st>>>(P.srec, P.inv, P.n, P.nwords, P.p, P.mask_bits, P.counts,
                                              P.codes, P.props);
  const int rc = check_launch("unsort");
  stage_mark(4, st);
  return rc;
}

int run_tile_path(TileParams P, const TileLayout& L, unsigned char* ws, const float* points,
                  int64_t n, cudaStream_t st) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws + L.keys);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  uint32_t* totals = reinterpret_cast<uint32_t*>(ws + L.totals);
  stage_mark(0, st);
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kSortBins, st);
  cudaMemsetAsync(P.ovf_count, 0, sizeof(int32_t), st);
  k_sort_keys<<<grid_for(n, 256), 256, 0, st>>>(points, n, P.lo_hi, keys, hist);
  if (int rc = check_launch("sort_keys")) return rc;
  k_scan_blocks<<<kSortBins / 4096, 1024, 0, st>>>(hist, totals);
  if (int rc = check_launch("scan_blocks")) return rc;
  k_scan_totals<<<1, 1024, 0, st>>>(totals, kSortBins / 4096);
  if (int rc = check_launch("scan_totals")) return rc;
  k_scan_add<<<kSortBins / 256, 256, 0, st>>>(hist, totals);
  if (int rc = check_launch("scan_add")) return rc;
  k_sort_scatter<<<grid_for(n, 256), 256, 0, st>>>(points, n, keys, hist, const_cast<int32_t*>(P.inv),
                                                   const_cast<float4*>(P.spts));
  if (int rc = check_launch("sort_scatter")) return rc;
  stage_mark(1, st);
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
  k_tile_prep<<<(unsigned)L.ntiles, kTile, 0, st>>>(Q);
  if (int rc = check_launch("tile_prep")) return rc;
  stage_mark(2, st);
  if (debug) {
    unsigned long long h[6];
    cudaMemcpyAsync(h, pdbg + 16 * 1000, sizeof(h), cudaMemcpyDeviceToHost, st);
    std::vector<int32_t> kt((size_t)L.ntiles);
    cudaMemcpyAsync(kt.data(), P.tile_kt, sizeof(int32_t) * kt.size(), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    double ksum = 0;
    int64_t over = 0, kmax = 0;
    for (int32_t k : kt) {
      ksum += k;
      over += ((k + 15) & ~15) > ws_kt_max();
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
    fprintf(stderr, "[prep debug] tile x view: FULL %.1f%%, MIXED %.1f%%, OFF %.1f%%; taps per tile mean %.1f "
            "max %lld, overflow tiles %lld of %lld\n", 100.0 * h[3] / h[5], 100.0 * h[4] / h[5],
            100.0 * (h[5] - h[3] - h[4]) / h[5], ksum / kt.size(), (long long)kmax, (long long)over,
            (long long)kt.size());
  }
  const int rc = run_tile_ws(P, st);
  stage_mark(3, st);
  return rc;
}

}  // namespace tile
}  // namespace pf

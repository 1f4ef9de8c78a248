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
// Kernels:
//   k_sort_keys / k_scan_* / k_sort_scatter — counting sort of the points by a 21-bit Morton key of
//       a 128^3 grid over the bbox (spatial coherence of tiles; no library sort);
//   k_tile_prep  — per tile: exact visibility (fp32 projection with a rigorous error bound, exact
//       fp64 fallback near any decision boundary -> bit-identical masks), counts, voxel codes, and
//       the per-view tap windows of the tile;
//   k_tile_mma   — per tile: build W in smem (K-major, 128-B swizzle), stream the taps' feature
//       rows chunk by chunk (cp.async, N-major swizzled), tcgen05.mma into TMEM, drain |F|^2, then
//       S = W . G and the epilogue. Tiles whose tap count exceeds KT_MAX fall back to the SIMT
//       kernel through an overflow list.
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
                               uint32_t* __restrict__ cursor, int32_t* __restrict__ perm,
                               float4* __restrict__ spts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t pos = atomicAdd(cursor + keys[i], 1u);
    perm[pos] = (int32_t)i;
    spts[pos] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2), 0.f);
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

// Tile-level occlusion cull for one view (exact): the tile's points lie in the box [lo, hi]; their
// camera depth is >= the minimum over the box corners (z is affine) and their pixels fall inside
// the projected corners' bounding rectangle (perspective maps a box in front of the camera into
// the convex hull of its projected corners). If every stored depth in that rectangle (+1 px) plus
// eps is below the box's minimum depth, no point of the tile can pass the depth test in this view
// (out-of-image and invalid pixels fail it anyway), so the per-point work is skipped.
__device__ bool tile_occluded(const ViewF& v, const float* __restrict__ depth, const float* lo,
                              const float* hi, float eps) {
  // fp32 with explicit slack: depths / pixels of the box corners are only used as conservative
  // bounds (+1e-5 m on the depth comparison, +1 px on the window), never as a visibility decision
  float zmin = 1e30f, umin = 1e30f, umax = -1e30f, vmin = 1e30f, vmax = -1e30f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float px = (c & 1) ? hi[0] : lo[0];
    const float py = (c & 2) ? hi[1] : lo[1];
    const float pz = (c & 4) ? hi[2] : lo[2];
    const float X = fmaf(v.R[2], pz, fmaf(v.R[1], py, v.R[0] * px)) + v.t[0];
    const float Y = fmaf(v.R[5], pz, fmaf(v.R[4], py, v.R[3] * px)) + v.t[1];
    const float Z = fmaf(v.R[8], pz, fmaf(v.R[7], py, v.R[6] * px)) + v.t[2];
    zmin = fminf(zmin, Z);
    const float rz = 1.f / Z;
    const float u = fmaf(v.fx, X * rz, v.cx), w = fmaf(v.fy, Y * rz, v.cy);
    umin = fminf(umin, u);
    umax = fmaxf(umax, u);
    vmin = fminf(vmin, w);
    vmax = fmaxf(vmax, w);
  }
  if (!(zmin > 1e-3f)) return false;
  if (umax < -2.f || vmax < -2.f || umin > (float)v.W + 1.f || vmin > (float)v.H + 1.f) return true;  // off-image
  const int x0 = max((int)floorf(umin) - 1, 0), x1 = min((int)ceilf(umax) + 1, v.W - 1);
  const int y0 = max((int)floorf(vmin) - 1, 0), y1 = min((int)ceilf(vmax) + 1, v.H - 1);
  if (x1 < x0 || y1 < y0) return true;
  if ((x1 - x0 + 1) * (y1 - y0 + 1) > 64) return false;
  const float* d = depth + v.depth_off + (int64_t)y0 * v.W + x0;
  float dmax0 = 0.f, dmax1 = 0.f;
  for (int y = 0; y <= y1 - y0; ++y, d += v.W) {
    int x = 0;
    for (; x + 1 <= x1 - x0; x += 2) {
      dmax0 = fmaxf(dmax0, __ldg(d + x));
      dmax1 = fmaxf(dmax1, __ldg(d + x + 1));
    }
    if (x <= x1 - x0) dmax0 = fmaxf(dmax0, __ldg(d + x));
  }
  return zmin - 1e-5f > fmaxf(dmax0, dmax1) + eps + 1e-5f;
}

__global__ void k_view_setup(TileParams P) {
  const int j = threadIdx.x;
  if (j < P.nv) {
    const ViewF w = make_viewf(P.views[j], P.d);
    P.viewf[j] = w;
    P.vbound[j] = view_bound(w, P.views[j], P.lo_hi);
  }
}

// ---- k_tile_prep ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kTile, 8) k_tile_prep(TileParams P) {
  __shared__ ViewF sv[kMaxViewsTC];
  __shared__ int wx0[kMaxViewsTC], wx1[kMaxViewsTC], wy0[kMaxViewsTC], wy1[kMaxViewsTC];
  __shared__ float4 sbound[kMaxViewsTC];  // per-view constant bounds: eu, ev, e, fast
  const int tid = threadIdx.x, lane = tid & 31;
  for (int j = tid; j < P.nv; j += kTile) {
    sv[j] = P.viewf[j];     // per-view fp32 camera + bounds computed once (k_view_setup)
    sbound[j] = P.vbound[j];
    wx0[j] = INT_MAX;
    wy0[j] = INT_MAX;
    wx1[j] = -1;
    wy1[j] = -1;
  }
  __syncthreads();
  const int64_t tile = blockIdx.x;
  const int64_t jpt = tile * kTile + tid;
  const bool valid = jpt < P.n;
  float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
  int32_t i = 0;
  if (valid) {
    p = P.spts[jpt];
    i = P.perm[jpt];
  }
  const float eps_f = (float)P.eps;
  // tile bbox -> per-view occlusion cull -> compact list of views that need per-point tests
  __shared__ float sbb[kTile / 32][6];
  __shared__ int s_views_list[kMaxViewsTC];
  __shared__ int s_nlist;
  {
    float b[6] = {valid ? p.x : INFINITY, valid ? p.y : INFINITY, valid ? p.z : INFINITY,
                  valid ? p.x : -INFINITY, valid ? p.y : -INFINITY, valid ? p.z : -INFINITY};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        b[a] = fminf(b[a], __shfl_xor_sync(0xffffffffu, b[a], o));
        b[a + 3] = fmaxf(b[a + 3], __shfl_xor_sync(0xffffffffu, b[a + 3], o));
      }
    }
    if (lane == 0)
#pragma unroll
      for (int a = 0; a < 6; ++a) sbb[tid >> 5][a] = b[a];
  }
  __syncthreads();
  __shared__ unsigned char s_keep[kMaxViewsTC];
  if (tid < P.nv) {
    float lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fminf(fminf(sbb[0][a], sbb[1][a]), fminf(sbb[2][a], sbb[3][a]));
      hi[a] = fmaxf(fmaxf(sbb[0][a + 3], sbb[1][a + 3]), fmaxf(sbb[2][a + 3], sbb[3][a + 3]));
    }
    s_keep[tid] = tile_occluded(sv[tid], P.depth, lo, hi, eps_f) ? 0 : 1;
  }
  __syncthreads();
  if (tid < 32) {  // ballot compaction of the kept views (<= 64: two per lane)
    const bool k0 = lane < P.nv && s_keep[lane], k1 = lane + 32 < P.nv && s_keep[lane + 32];
    const uint32_t b0 = __ballot_sync(0xffffffffu, k0), b1 = __ballot_sync(0xffffffffu, k1);
    const uint32_t below = (1u << lane) - 1u;
    if (k0) s_views_list[__popc(b0 & below)] = lane;
    if (k1) s_views_list[__popc(b0) + __popc(b1 & below)] = lane + 32;
    const int n = __popc(b0) + __popc(b1);
    if (lane == 0) s_nlist = n;
    if (P.dbg && lane == 0) {
      atomicAdd(P.dbg + 16 * 1000 + 3, (unsigned long long)n);
      atomicAdd(P.dbg + 16 * 1000 + 4, (unsigned long long)P.nv);
    }
  }
  __syncthreads();
  const int nlist = s_nlist;
  uint32_t words[kMaxViewsTC / 32] = {0u, 0u};
  int cnt = 0;
  constexpr int U = 4;  // views in flight per thread (independent depth loads)
  for (int l0 = 0; l0 < nlist; l0 += U) {
    ProjF q[U];
    int st[U];
    float stored[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      st[u] = kInvisible;
      stored[u] = 0.f;
      const int v = l0 + u < nlist ? s_views_list[l0 + u] : 0;
      if (valid && l0 + u < nlist) {
        q[u] = project_f32(sv[v], p.x, p.y, p.z);
        int64_t didx = 0;
        const float4 b = sbound[v];
        st[u] = b.w > 0.f ? classify_fast(sv[v], b, q[u], didx) : classify(sv[v], q[u], didx);
        if (st[u] == kNeedDepth) stored[u] = __ldg(P.depth + didx);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (l0 + u >= nlist) break;
      const int v = s_views_list[l0 + u];
      int s = st[u];
      if (s == kNeedDepth) s = depth_decide(q[u], stored[u], eps_f);
      bool vis = s == kNeedDepth;
      if (s == kAmbiguous) vis = visible_f64(P.views[v], P.depth, p.x, p.y, p.z, P.eps);  // rare
      if (P.dbg) {  // PF_WS_DEBUG: fraction of samples decided in fp64 / warp-iterations with any
        const unsigned amb = __ballot_sync(0xffffffffu, s == kAmbiguous);
        if (lane == 0) {
          atomicAdd(P.dbg + 16 * 1000, (unsigned long long)__popc(amb));
          atomicAdd(P.dbg + 16 * 1000 + 1, (unsigned long long)(amb != 0u));
          atomicAdd(P.dbg + 16 * 1000 + 2, 1ull);
        }
      }
      if (__any_sync(0xffffffffu, vis)) {
        int tx0 = INT_MAX, ty0 = INT_MAX, tx1 = -1, ty1 = -1;
        if (vis) {
          const TapF t = taps_f32(sv[v], q[u].u, q[u].v);
          tx0 = t.x0;
          ty0 = t.y0;
          tx1 = t.x0 + t.dx;
          ty1 = t.y0 + t.dy;
          words[v >> 5] |= 1u << (v & 31);
          ++cnt;
        }
        const int ax0 = __reduce_min_sync(0xffffffffu, tx0), ay0 = __reduce_min_sync(0xffffffffu, ty0);
        const int ax1 = __reduce_max_sync(0xffffffffu, tx1), ay1 = __reduce_max_sync(0xffffffffu, ty1);
        if (lane == 0) {
          atomicMin(wx0 + v, ax0);
          atomicMin(wy0 + v, ay0);
          atomicMax(wx1 + v, ax1);
          atomicMax(wy1 + v, ay1);
        }
      }
    }
  }
  if (valid) {
    for (int w = 0; w < P.nwords; ++w) P.mask_bits[(int64_t)i * P.nwords + w] = words[w];
    P.counts[i] = cnt;
    double lo[3];
    const double edge = voxel_edge(P.lo_hi, P.grid, lo);
    P.codes[i] = voxel_code(p.x, p.y, p.z, lo, edge, P.grid);
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
      sz[r] = w[r] * h[r];
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


// ---- k_tile_mma ----------------------------------------------------------------------------------------
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

__global__ void __launch_bounds__(kTile, 2) k_tile_mma(TileParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;                            // 128 x KT_MAX bf16, K-major SW128
  unsigned char* sB = smem + kTile * kKtMax * 2;       // 2 stages x (KT_MAX x 64) bf16, N-major SW128
  float* sRed = reinterpret_cast<float*>(smem);        // epilogue: [128][kRedStride] (reuses A+B)
  __shared__ ViewF sv[kMaxViewsTC];
  __shared__ uint2 sdesc[kMaxViewsTC];
  __shared__ int32_t scell[kKtMax];
  __shared__ __align__(16) float svals[kMaxKpadTC * 4];
  __shared__ float smt[kMaxKpadTC];
  __shared__ float srs[kTile];
  __shared__ float sred6[4][8];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ int s_kt;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tile = blockIdx.x;
  if (tid == 0) s_kt = P.tile_kt[tile];
  for (int j = tid; j < P.nv; j += kTile) {
    sv[j] = make_viewf(P.views[j], P.d);
    sdesc[j] = P.tile_desc[tile * P.nv + j];
  }
  for (int j = tid; j < P.kpadg * 4; j += kTile) {
    const int kk = j >> 2, pp = j & 3;
    svals[j] = (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f;
  }
  for (int j = tid; j < P.kpadg; j += kTile) smt[j] = j < P.k ? P.mid_theta[j] : 0.f;
  __syncthreads();
  const int kt = s_kt;
  const int ktp = (kt + 15) & ~15;
  const int64_t jpt = tile * kTile + tid;
  const bool valid = jpt < P.n;
  const int32_t i = valid ? P.perm[jpt] : 0;
  if (ktp > kKtMax || kt == 0) {
    // overflow (or nothing visible anywhere in the tile): the SIMT kernel handles these points
    if (valid) P.ovf_list[atomicAdd(P.ovf_count, 1)] = i;
    for (int kk = tid; kk < P.k + 6; kk += kTile) P.tile_part[tile * (int64_t)(P.k + 6) + kk] = 0.f;
    return;
  }
  const float4 p = valid ? P.spts[jpt] : make_float4(0.f, 0.f, 0.f, 0.f);

  // row -> global cell table for the B loads (pad rows repeat a valid cell; their A columns are 0)
  for (int v = tid; v < P.nv; v += kTile) {
    const uint2 ds = sdesc[v];
    const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
    const int w = ds.y & 0xff, h = (ds.y >> 8) & 0xff;
    for (int a = 0; a < w * h; ++a)
      scell[base + a] = sv[v].cell_base + (y0 + a / w) * sv[v].Wf + x0 + a % w;
  }
  // zero A: ceil(ktp/64) atom columns of [128 rows][128 B]
  {
    uint4* a4 = reinterpret_cast<uint4*>(sA);
    for (int e = tid; e < ((ktp + 63) >> 6) * kTile * 8; e += kTile) a4[e] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  for (int r = ktp - 1 - tid; r >= kt; r -= kTile) scell[r] = scell[0];
  __syncthreads();

  // chunk schedule: nd feature chunks of 64 channels (TMEM D double buffer), then ns S chunks
  const int nd = P.d >> 6;
  const int ns = (P.kpadg + 63) >> 6;
  const int nch = nd + ns;
  auto chunk_cols = [&](int c) { return c < nd ? 64 : min(64, P.kpadg - 64 * (c - nd)); };
  // B loader: thread -> fixed 16-byte column q, rows r0, r0 + rstep, ...
  auto issue_load = [&](int c) {
    const int ncol = chunk_cols(c);
    const int qn = ncol >> 3;  // 8 or 4 (power of two)
    const int q = tid & (qn - 1);
    const int rstep = kTile / qn;
    unsigned char* stage = sB + (c & 1) * (kKtMax * 128);
    const uint16_t* base;
    int64_t rowlen;
    if (c < nd) {
      base = reinterpret_cast<const uint16_t*>(P.fmap) + c * 64 + q * 8;
      rowlen = P.d;
    } else {
      base = P.Gbf + (c - nd) * 64 + q * 8;
      rowlen = P.kpadg;
    }
    const uint32_t sbase = tc::smem_u32(stage);
    for (int r = tid / qn; r < ktp; r += rstep)
      tc::cp_async16(sbase + tc::b_chunk_off(r, q, ktp), base + (int64_t)scell[r] * rowlen);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue_load(0);

  // scatter this point's bilinear weights into its A row (overlaps the first B load)
  int count = 0;
  if (valid) {
    count = P.counts[i];
    for (int w = 0; w < P.nwords; ++w) {
      uint32_t bits = P.mask_bits[(int64_t)i * P.nwords + w];
      while (bits) {
        const int v = w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
        const ProjF q = project_f32(sv[v], p.x, p.y, p.z);
        const TapF t = taps_f32(sv[v], q.u, q.v);
        float w00 = (1.f - t.wy) * (1.f - t.wx), w01 = (1.f - t.wy) * t.wx;
        float w10 = t.wy * (1.f - t.wx), w11 = t.wy * t.wx;
        if (!t.dx) { w00 += w01; w10 += w11; }
        if (!t.dy) { w00 += w10; w01 += w11; }
        const uint2 ds = sdesc[v];
        const int base = ds.x & 0xffff, x0 = (ds.x >> 16) & 0xff, y0 = ds.x >> 24;
        const int ww = ds.y & 0xff;
        const int c00 = base + (t.y0 - y0) * ww + (t.x0 - x0);
        *reinterpret_cast<uint16_t*>(sA + tc::a_off(tid, c00, kTile)) = f2bf(w00);
        if (t.dx) *reinterpret_cast<uint16_t*>(sA + tc::a_off(tid, c00 + 1, kTile)) = f2bf(w01);
        if (t.dy) *reinterpret_cast<uint16_t*>(sA + tc::a_off(tid, c00 + ww, kTile)) = f2bf(w10);
        if (t.dx && t.dy) *reinterpret_cast<uint16_t*>(sA + tc::a_off(tid, c00 + ww + 1, kTile)) = f2bf(w11);
      }
    }
  }
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
  }
  const uint32_t ncols = P.tmem_cols;
  if (warp == 0) tc::tmem_alloc(&tmem_base_s, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = tmem_base_s;
  const uint32_t t_lane = (uint32_t)(warp * 32) << 16;
  const uint32_t tS = tbase + 128;
  const float invc = count > 0 ? 1.f / (float)count : 0.f;
  float ss = 0.f;

  auto drain = [&](int c) {  // |F|^2 (and optional mean features) from TMEM D buffer c & 1
    const uint32_t tD = tbase + (uint32_t)((c & 1) * 64);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tD + t_lane + c0, v);
#pragma unroll
      for (int q = 0; q < 32; ++q) ss = fmaf(v[q], v[q], ss);
      if (P.features && valid) {
        float* dst = P.features + (int64_t)i * P.d + c * 64 + c0;
#pragma unroll
        for (int q = 0; q < 32; q += 4)
          *reinterpret_cast<float4*>(dst + q) =
              make_float4(v[q] * invc, v[q + 1] * invc, v[q + 2] * invc, v[q + 3] * invc);
      }
    }
  };

  for (int c = 0; c < nch; ++c) {
    // B(c) landed (only chunk c+1's group may still be in flight... it is issued below)
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    tc::fence_async_shared();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
      const int ncol = chunk_cols(c);
      const uint32_t idesc = tc::idesc_bf16_f32(128, ncol, false, true);
      const uint32_t a0 = tc::smem_u32(sA), b0 = tc::smem_u32(sB + (c & 1) * (kKtMax * 128));
      const uint32_t dst = c < nd ? tbase + (uint32_t)((c & 1) * 64) : tS + (uint32_t)(64 * (c - nd));
      for (int s = 0; s < ktp / 16; ++s) {
        const uint64_t ad = tc::smem_desc_sw128(a0 + (s >> 2) * kTile * 128 + (s & 3) * 32, 16, 1024);
        const uint64_t bd = tc::smem_desc_sw128(b0 + s * 2048, ktp * 128, 1024);
        tc::mma_bf16(dst, ad, bd, idesc, s > 0 ? 1u : 0u);
      }
      tc::mma_commit(&mbar[c & 1]);
    }
    if (c >= 1) {
      tc::mbar_wait(&mbar[(c - 1) & 1], ((c - 1) >> 1) & 1);
      tc::fence_after_sync();
      if (c - 1 < nd) drain(c - 1);
    }
    // stage (c+1)&1 was read by MMA c-1, which has completed (waited above by every thread)
    if (c + 1 < nch) issue_load(c + 1);
  }
  tc::mbar_wait(&mbar[(nch - 1) & 1], ((nch - 1) >> 1) & 1);
  tc::fence_after_sync();
  if (nch - 1 < nd) drain(nch - 1);

  // ---- epilogue: thread = point; S row in TMEM -----------------------------------------------------
  const bool featured = valid && count > 0;
  const float inv = ss > 0.f ? 1.f / sqrtf(ss) : 0.f;
  const float sc = inv * P.inv_temp * 1.4426950408889634f;  // log2(e) * inv / T
  float m2 = -INFINITY;                                      // max of s * log2(e) / T
  bool nan = false;
  for (int c0 = 0; c0 < P.kpadg; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tS + t_lane + c0, v);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const float x = v[q] * sc;
      if (c0 + q < P.k) {
        nan |= isnan(x);
        m2 = fmaxf(m2, x);
      }
    }
  }
  if (featured && nan) atomicOr(P.status, 1);
  float se = 0.f, pl0 = 0.f, pl1 = 0.f, pl2 = 0.f, pl3 = 0.f, pml = 0.f;
  const float4* sv4 = reinterpret_cast<const float4*>(svals);
  for (int c0 = 0; c0 < P.kpadg; c0 += 32) {
    float v[32];
    tc::tmem_ld32(tS + t_lane + c0, v);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int kk = c0 + q;
      const float e = kk < P.k ? exp2f(v[q] * sc - m2) : 0.f;
      se += e;
      const float4 y = sv4[kk];
      pl0 = fmaf(e, y.x, pl0);
      pl1 = fmaf(e, y.y, pl1);
      pl2 = fmaf(e, y.z, pl2);
      pl3 = fmaf(e, y.w, pl3);
      pml = fmaf(e, smt[kk], pml);
      sRed[tid * kRedStride + kk] = e;
    }
  }
  const float rs = featured ? 1.f / se : 0.f;
  srs[tid] = rs;
  if (P.sims || P.weights) {  // validation outputs (uniform branch)
    for (int c0 = 0; c0 < P.kpadg; c0 += 32) {
      float v[32];
      tc::tmem_ld32(tS + t_lane + c0, v);
      if (valid) {
        for (int q = 0; q < 32 && c0 + q < P.k; ++q) {
          if (P.sims) P.sims[(int64_t)i * P.k + c0 + q] = featured ? v[q] * inv : 0.f;
          if (P.weights) P.weights[(int64_t)i * P.k + c0 + q] = sRed[tid * kRedStride + c0 + q] * rs;
        }
      }
    }
  }
  const float prop[4] = {pl0 * rs, pl1 * rs, pl2 * rs, pl3 * rs};
  const float pm = pml * rs;
  if (valid) {
    for (int pp = 0; pp < P.p; ++pp) P.props[(int64_t)i * P.p + pp] = prop[pp];
    if (P.grid_partials) {
      const int32_t code = P.codes[i];
      atomicAdd(P.grid_partials + code, prop[P.density_col]);
      atomicAdd(P.grid_partials + P.cells3 + code, 1.0f);
    }
  }
  // block partials: weight totals = column sums of e * rs, scalars by warp + block reduction
  float r6[6] = {pm, pm * p.x, pm * p.y, pm * p.z, featured ? 1.f : 0.f, (float)count};
#pragma unroll
  for (int q = 0; q < 6; ++q) r6[q] = warp_sum(r6[q]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 6; ++q) sred6[warp][q] = r6[q];
  tc::fence_before_sync();
  __syncthreads();
  float* out = P.tile_part + tile * (int64_t)(P.k + 6);
  for (int kk = tid; kk < P.k; kk += kTile) {
    float acc = 0.f;
#pragma unroll 8
    for (int r = 0; r < kTile; ++r) acc = fmaf(sRed[r * kRedStride + kk], srs[r], acc);
    out[kk] = acc;
  }
  if (tid < 6) out[P.k + tid] = sred6[0][tid] + sred6[1][tid] + sred6[2][tid] + sred6[3][tid];
  if (warp == 0) tc::tmem_dealloc(tbase, ncols);
}


__global__ void k_tile_partials(const float* __restrict__ tile_part, int64_t ntiles, int ncol,
                                double* __restrict__ partials) {
  const int col = threadIdx.x;
  if (col >= ncol) return;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
  double acc = 0.0;
  for (int64_t t = t0; t < t1; ++t) acc += (double)tile_part[t * ncol + col];
  if (acc != 0.0) atomicAdd(partials + col, acc);
}

// G in bf16 (cells x kpadg) for the tensor path, from the fp32 table of the SIMT path
__global__ void k_g_bf16(const float* __restrict__ G, int64_t cells, int kpad, int kpadg,
                         uint16_t* __restrict__ Gbf) {
  const int64_t total = cells * kpadg;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / kpadg;
    const int k = (int)(e - c * kpadg);
    Gbf[e] = f2bf(k < kpad ? G[c * kpad + k] : 0.f);
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
  L.perm = take(sizeof(int32_t) * (size_t)n);
  L.spts = take(sizeof(float4) * (size_t)n);
  L.desc = take(sizeof(uint2) * (size_t)ntiles * nv);
  L.kt = take(sizeof(int32_t) * (size_t)ntiles);
  L.part = take(sizeof(float) * (size_t)ntiles * (kMaxKpadTC + 6));
  L.viewf = take(sizeof(ViewF) * kMaxViewsTC);
  L.vbound = take(sizeof(float4) * kMaxViewsTC);
  L.ovf = take(sizeof(int32_t) * (size_t)(n + 1));
  L.gbf = take(sizeof(uint16_t) * (size_t)cells * kpadg);
  L.bytes = off;
  return L;
}

size_t tile_smem_bytes() {
  const size_t ab = (size_t)kTile * kKtMax * 2 * 2;
  const size_t red = (size_t)kTile * kRedStride * 4;
  return (ab > red ? ab : red) + 1024;
}

int run_g_bf16(const float* G, int64_t cells, int kpad, int kpadg, uint16_t* Gbf, cudaStream_t st) {
  k_g_bf16<<<grid_for(cells * kpadg, 256), 256, 0, st>>>(G, cells, kpad, kpadg, Gbf);
  return check_launch("g_bf16");
}

int run_tile_path(TileParams P, const TileLayout& L, unsigned char* ws, const float* points,
                  int64_t n, int64_t cells, const float* G, int kpad, int hf, int wf, cudaStream_t st) {
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws + L.keys);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  uint32_t* totals = reinterpret_cast<uint32_t*>(ws + L.totals);
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
  k_sort_scatter<<<grid_for(n, 256), 256, 0, st>>>(points, n, keys, hist, const_cast<int32_t*>(P.perm),
                                                   const_cast<float4*>(P.spts));
  if (int rc = check_launch("sort_scatter")) return rc;
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
  if (debug) {
    unsigned long long h[5];
    cudaMemcpyAsync(h, pdbg + 16 * 1000, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[prep debug] ambiguous samples %.4f%%, warp-iterations with any %.2f%%, views kept "
            "after the tile cull %.1f%%\n", 100.0 * h[0] / (32.0 * h[2]), 100.0 * h[1] / h[2],
            100.0 * h[3] / h[4]);
  }
  if (int rc = check_launch("tile_prep")) return rc;
  // persistent warp-specialised TMA kernel (pf_tile_ws.cu); k_tile_mma when TMA maps are unavailable
  static const bool force_v2 = getenv("PF_TILE_KERNEL") && !strcmp(getenv("PF_TILE_KERNEL"), "v2");
  if (!force_v2) {
    const int rc = run_tile_ws(P, hf, wf, P.nv, st);
    if (rc >= 0) return rc;
  }
  const size_t smem = tile_smem_bytes();
  cudaFuncSetAttribute(k_tile_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tile_mma<<<(unsigned)L.ntiles, kTile, smem, st>>>(P);
  if (int rc = check_launch("tile_mma")) return rc;
  const int ncol = P.k + 6;
  k_tile_partials<<<256, ((ncol + 31) / 32) * 32, 0, st>>>(P.tile_part, L.ntiles, ncol, P.partials);
  return check_launch("tile_partials");
}

}  // namespace tile
}  // namespace pf

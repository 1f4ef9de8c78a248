// Device helpers shared by the tile-path kernels (pf_tile.cu, pf_tile_ws.cu): the fp32 projection
// with its rigorous error bound, the exact visibility decision and the bilinear tap geometry.
#pragma once

#include "pf_common.cuh"
#include "pf_tile.cuh"

namespace pf {
namespace tile {

// order-preserving float <-> int keys (signed compare), for warp min / max bounds with one REDUX
__device__ __forceinline__ int float_key(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float key_float(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// ---- fp32 projection with a rigorous error bound ----------------------------------------------------
__device__ __forceinline__ ViewF make_viewf(const pf_view_t& v, int d) {
  ViewF w;
#pragma unroll
  for (int q = 0; q < 9; ++q) w.R[q] = (float)v.R[q];
  w.t[0] = (float)v.t[0];
  w.t[1] = (float)v.t[1];
  w.t[2] = (float)v.t[2];
  w.fx = (float)v.fx;
  w.fy = (float)v.fy;
  w.cx = (float)v.cx;
  w.cy = (float)v.cy;
  w.ru = (float)((double)v.Wf / (double)v.W);
  w.rv = (float)((double)v.Hf / (double)v.H);
  w.tmax = fmaxf(fmaxf(fabsf(w.t[0]), fabsf(w.t[1])), fabsf(w.t[2]));
  w.H = v.H;
  w.W = v.W;
  w.Hf = v.Hf;
  w.Wf = v.Wf;
  w.cell_base = (int32_t)(v.fmap_offset / d);
  w.depth_off = v.depth_offset;
  return w;
}

struct ProjF {
  float u, v, z, e;  // e: bound on |cam_c - cam_c(exact)| for each camera coordinate
  float X, Y, rz;    // camera x, y and the rounded reciprocal of z
};

__device__ __forceinline__ float cam_f32(const float* R, float t, float px, float py, float pz) {
  return __fadd_rn(__fmaf_rn(R[2], pz, __fmaf_rn(R[1], py, __fmul_rn(R[0], px))), t);
}

// u = fx * (X * (1/z)) + cx with explicitly rounded ops (k_tile_prep and k_tile_mma must agree
// bit for bit, so nothing is left to contraction choices)
__device__ __forceinline__ ProjF project_f32(const ViewF& w, float px, float py, float pz) {
  ProjF o;
  o.X = cam_f32(w.R + 0, w.t[0], px, py, pz);
  o.Y = cam_f32(w.R + 3, w.t[1], px, py, pz);
  o.z = cam_f32(w.R + 6, w.t[2], px, py, pz);
  o.rz = __frcp_rn(o.z);
  o.u = __fmaf_rn(w.fx, __fmul_rn(o.X, o.rz), w.cx);
  o.v = __fmaf_rn(w.fy, __fmul_rn(o.Y, o.rz), w.cy);
  // |R_ij| <= 1: each camera coordinate has magnitude <= |p|_1 + |t|_inf. f32 R/t representation
  // (2^-24 relative) plus 4 roundings of that magnitude is < 5*2^-24; take 2^-21 (1.6x margin).
  o.e = (fabsf(px) + fabsf(py) + fabsf(pz) + w.tmax) * 4.76837158203125e-07f;
  return o;
}

// Bound on |u - u64| for u = f * num/z + c, given |num - num*|, |z - z*| <= e and |z| >= 2e:
// |a - a*| <= e/|z| + e(|num| + e)/z^2 (taken twice) + 2^-23|a| (rcp + mul roundings); the fma adds
// 2^-24 |f a + c| and f / c representation 2^-24 each (taken as 2^-23). No divisions.
__device__ __forceinline__ float pix_err(float f, float c, float num, float arz, float e) {
  const float a = fabsf(num) * arz;
  const float da = e * arz * (1.f + 2.f * (fabsf(num) + e) * arz) + 1.2e-7f * a;
  return fabsf(f) * da + 1.2e-7f * (fabsf(f) * a + fabsf(c)) + 1e-6f;
}

// Classification of one (point, view) sample before the depth lookup.
enum : int { kInvisible = 0, kNeedDepth = 1, kAmbiguous = 2 };

__device__ __forceinline__ int classify(const ViewF& w, const ProjF& q, int64_t& didx) {
  const float e = q.e;
  if (!(fabsf(q.z) > 2.f * e) || !isfinite(q.u) || !isfinite(q.v)) return kAmbiguous;
  if (q.z < 0.f) return kInvisible;  // |z| > 2e: the sign is certain
  const float arz = fabsf(q.rz) * 1.0000005f;
  const float eu = pix_err(w.fx, w.cx, q.X, arz, e);
  const float ev = pix_err(w.fy, w.cy, q.Y, arz, e);
  const float du = fabsf(q.u - floorf(q.u) - 0.5f), dv = fabsf(q.v - floorf(q.v) - 0.5f);
  if (eu >= 0.25f || ev >= 0.25f || du <= eu || dv <= ev) return kAmbiguous;
  const float ru = rintf(q.u), rv = rintf(q.v);
  if (!(ru >= 0.f && ru < (float)w.W && rv >= 0.f && rv < (float)w.H)) return kInvisible;
  didx = w.depth_off + (int64_t)rv * w.W + (int64_t)ru;
  return kNeedDepth;
}

// depth test for a decided pixel: z64 <= stored + eps (f64) decided in f32 with margin
__device__ __forceinline__ int depth_decide(const ProjF& q, float stored, float eps_f) {
  if (!(stored > 0.f)) return kInvisible;
  const float thr = __fadd_rn(stored, eps_f);
  const float m = q.e + 2.4e-7f * fabsf(thr) + 1e-9f;
  if (q.z + m < thr) return kNeedDepth;  // visible
  if (q.z - m > thr) return kInvisible;
  return kAmbiguous;
}

// exact fp64 decision, identical to the reference arithmetic (pf_common.cuh)
__device__ __forceinline__ bool visible_f64(const pf_view_t& w64, const float* depth, float px,
                                            float py, float pz, double eps) {
  const Proj p64 = project(w64, (double)px, (double)py, (double)pz);
  return depth_test(depth + w64.depth_offset, w64.H, w64.W, p64.u, p64.v, p64.z, eps);
}


// bilinear taps of a visible sample from the fp32 projection (fusion.py:83-86 +
// numpy_impl.py:50-57); k_tile_prep and k_tile_mma call this with bit-identical inputs.
__device__ __forceinline__ TapF taps_f32(const ViewF& w, float u, float v) {
  TapF t;
  const float fu = __fsub_rn(__fmul_rn(__fadd_rn(u, 0.5f), w.ru), 0.5f);
  const float fv = __fsub_rn(__fmul_rn(__fadd_rn(v, 0.5f), w.rv), 0.5f);
  const float x = fminf(fmaxf(fu, 0.f), (float)(w.Wf - 1));
  const float y = fminf(fmaxf(fv, 0.f), (float)(w.Hf - 1));
  const float x0 = floorf(x), y0 = floorf(y);
  t.x0 = (int)x0;
  t.y0 = (int)y0;
  t.dx = t.x0 < w.Wf - 1 ? 1 : 0;
  t.dy = t.y0 < w.Hf - 1 ? 1 : 0;
  t.wx = __fsub_rn(x, x0);
  t.wy = __fsub_rn(y, y0);
  return t;
}

}  // namespace tile
}  // namespace pf

// Shared device helpers for the propfield B200 kernels (sm_100a).
//
// The fp64 projection helpers reproduce the reference's numpy arithmetic bit for bit:
// `cam = p @ R.T + t` (geometry.py:54) is an OpenBLAS dgemm whose per-element result is
// fma(p2,R[.,2], fma(p1,R[.,1], p0*R[.,0])) + t (pinned by tests/test_oracle.py::
// TestProjectionOperationOrder against this image's numpy), and
// `u = fx * X / z + cx` (geometry.py:57-58) is three separately rounded ops. Explicit __fma_rn /
// __dmul_rn / __ddiv_rn / __dadd_rn intrinsics stop nvcc from contracting or reordering them.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/propfield_b200.h"

namespace pf {

// PF_CHECK builds (nvcc -DPF_CHECK): device-side bounds checks on the indexed accesses of the tile
// path (gathered tap rows, window slots, sorted-record rows, work-list slots); a violation prints
// its site and traps, turning a silent out-of-bounds access into a launch error. The substitute for
// compute-sanitizer memcheck, which is closed on this pool.
#ifdef PF_CHECK
#define PF_DCHECK(cond, what)                                                                          \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("PF_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                        \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define PF_DCHECK(cond, what) \
  do {                        \
  } while (0)
#endif

constexpr int kWarp = 32;

// ---- host-side status plumbing (defined in pf_host.cu) ---------------------------------------
int set_error(int status, const char* fmt, ...);
int check_launch(const char* what);
void note_launch();
// stage timer marks of the tile path: 0 start, 1 sorted, 2 prepped, 3 tile kernel, 4 unsorted,
// 5 overflow done (pf_stage_timing / pf_stage_times)
constexpr int kStageMarks = 6;
void stage_mark(int mark, cudaStream_t st);

// ---- fp64 projection matching numpy ------------------------------------------------------------
struct Proj {
  double u, v, z;
};

__device__ __forceinline__ double cam_row(const double* R, int r, double px, double py, double pz,
                                          double t) {
  // numpy matmul (OpenBLAS dgemm small kernel): fma chain in column order, then + t.
  double acc = __dmul_rn(px, R[3 * r + 0]);
  acc = __fma_rn(py, R[3 * r + 1], acc);
  acc = __fma_rn(pz, R[3 * r + 2], acc);
  return __dadd_rn(acc, t);
}

__device__ __forceinline__ Proj project(const pf_view_t& vw, double px, double py, double pz) {
  Proj o;
  const double X = cam_row(vw.R, 0, px, py, pz, vw.t[0]);
  const double Y = cam_row(vw.R, 1, px, py, pz, vw.t[1]);
  o.z = cam_row(vw.R, 2, px, py, pz, vw.t[2]);
  o.u = __dadd_rn(__ddiv_rn(__dmul_rn(vw.fx, X), o.z), vw.cx);
  o.v = __dadd_rn(__ddiv_rn(__dmul_rn(vw.fy, Y), o.z), vw.cy);
  return o;
}

// numpy_impl.visible_in_view (numpy_impl.py:31-40): rint is round-half-even, matching np.rint.
__device__ __forceinline__ bool depth_test(const float* __restrict__ depth, int h, int w, double u,
                                           double v, double z, double eps) {
  if (!(z > 0.0)) return false;
  const double ru = rint(u), rv = rint(v);
  // compare in double before converting: huge / NaN pixels are simply out of bounds
  if (!(ru >= 0.0 && ru < (double)w && rv >= 0.0 && rv < (double)h)) return false;
  const int iu = (int)ru, iv = (int)rv;
  const double stored = (double)__ldg(depth + (int64_t)iv * w + iu);
  return stored > 0.0 && z <= __dadd_rn(stored, eps);
}

// fusion.py:83-86: fu = (u + 0.5) * (wf / w) - 0.5 with (wf / w) a separately rounded quotient.
__device__ __forceinline__ double feat_coord(double u, double ratio) {
  return __dsub_rn(__dmul_rn(__dadd_rn(u, 0.5), ratio), 0.5);
}

// bilinear tap geometry of numpy_impl.bilinear_gather (numpy_impl.py:50-57)
struct Taps {
  int x0, x1, y0, y1;
  double wx, wy;
};

__device__ __forceinline__ Taps make_taps(double fu, double fv, int hf, int wf) {
  Taps t;
  const double x = fmin(fmax(fu, 0.0), (double)wf - 1.0);
  const double y = fmin(fmax(fv, 0.0), (double)hf - 1.0);
  const double fx0 = floor(x), fy0 = floor(y);
  t.x0 = (int)fx0;
  t.y0 = (int)fy0;
  t.x1 = min(t.x0 + 1, wf - 1);
  t.y1 = min(t.y0 + 1, hf - 1);
  t.wx = __dsub_rn(x, fx0);
  t.wy = __dsub_rn(y, fy0);
  return t;
}

// ---- feature loads -------------------------------------------------------------------------------
__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

template <int DT>
__device__ __forceinline__ float load_feat(const void* base, int64_t idx) {
  if constexpr (DT == PF_F32) {
    return __ldg(reinterpret_cast<const float*>(base) + idx);
  } else {
    return bf16_bits_to_f32(__ldg(reinterpret_cast<const unsigned short*>(base) + idx));
  }
}

// ---- warp reductions ---------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// order-preserving float <-> uint mapping for atomicMin/Max on floats
__device__ __forceinline__ uint32_t float_flip(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__host__ __device__ __forceinline__ float float_unflip(uint32_t u) {
  u = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}

// ---- voxel indexing (sampling.py:110-123 convention) -------------------------------
__device__ __forceinline__ double voxel_edge(const double* lo_hi, int g, double lo[3]) {
  lo[0] = lo_hi[0];
  lo[1] = lo_hi[1];
  lo[2] = lo_hi[2];
  const double ext = fmax(fmax(__dsub_rn(lo_hi[3], lo[0]), __dsub_rn(lo_hi[4], lo[1])),
                          __dsub_rn(lo_hi[5], lo[2]));
  return __ddiv_rn(ext, (double)g);
}

__device__ __forceinline__ int voxel_axis(float p, double lo, double edge, int g) {
  if (!(edge > 0.0)) return 0;  // degenerate (single-point) domain: one voxel
  const double f = floor(__ddiv_rn(__dsub_rn((double)p, lo), edge));
  return (int)fmin(fmax(f, 0.0), (double)(g - 1));
}

__device__ __forceinline__ int32_t voxel_code(float x, float y, float z, const double lo[3],
                                              double edge, int g) {
  const int cx = voxel_axis(x, lo[0], edge, g);
  const int cy = voxel_axis(y, lo[1], edge, g);
  const int cz = voxel_axis(z, lo[2], edge, g);
  return (cx * g + cy) * g + cz;
}

inline int grid_for(int64_t work, int block, int max_blocks = 148 * 16) {
  int64_t g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (int)g;
}

}  // namespace pf

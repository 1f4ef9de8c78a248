// Voxel-grid mass (BASELINE-defined) and the object bbox that fixes its domain.
//
// Indexing follows the only voxel convention in the reference, sampling.py:110-123
// (`cell = floor((p - lo) / edge)`, clipped onto the grid, `code = (cx*G + cy)*G + cz`), with
// lo = per-axis min and edge = max extent / G. The index math is fp64 with explicitly rounded ops
// so codes are bit-exact with the numpy oracle. Occupancy is a 1-voxel shell: a voxel is occupied
// iff >= 1 point falls in it; mass = edge^3 * sum_occupied mean(rho).
#include "pf_common.cuh"

namespace pf {
namespace {

__global__ void k_bbox_init(uint32_t* s) {
  if (threadIdx.x < 3) s[threadIdx.x] = 0xffffffffu;      // min of flipped
  else if (threadIdx.x < 6) s[threadIdx.x] = 0u;          // max of flipped
}

__global__ void k_bbox_reduce(const float* __restrict__ p, int64_t n, uint32_t* __restrict__ s) {
  uint32_t mn[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, mx[3] = {0u, 0u, 0u};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint32_t f = float_flip(__ldg(p + 3 * i + a));
      mn[a] = min(mn[a], f);
      mx[a] = max(mx[a], f);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
      mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(s + a, mn[a]);
      atomicMax(s + 3 + a, mx[a]);
    }
  }
}

__global__ void k_bbox_final(double* lo_hi) {
  const uint32_t* s = reinterpret_cast<const uint32_t*>(lo_hi);
  uint32_t v[6];
#pragma unroll
  for (int a = 0; a < 6; ++a) v[a] = s[a];
#pragma unroll
  for (int a = 0; a < 6; ++a) lo_hi[a] = (double)float_unflip(v[a]);
}

__global__ void k_codes(const float* __restrict__ p, int64_t n, const double* __restrict__ lo_hi,
                        int g, int32_t* __restrict__ codes) {
  double lo[3];
  const double edge = voxel_edge(lo_hi, g, lo);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    codes[i] = voxel_code(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2), lo, edge, g);
}

__global__ void k_vox_acc(const int32_t* __restrict__ codes, const float* __restrict__ rho,
                          int64_t n, int64_t cells, float* __restrict__ grid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = codes[i];
    atomicAdd(grid + c, rho[i]);
    atomicAdd(grid + cells + c, 1.0f);
  }
}

__global__ void k_vox_mass(const float* __restrict__ grid, int64_t cells, double* __restrict__ out) {
  double acc = 0.0, occ = 0.0;
  const float4* s4 = reinterpret_cast<const float4*>(grid);
  const float4* c4 = reinterpret_cast<const float4*>(grid + cells);
  const int64_t n4 = (cells % 4 == 0) ? cells / 4 : 0;  // float4 view needs 16-byte alignment
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 c = __ldcs(c4 + i);
    if (c.x + c.y + c.z + c.w > 0.0f) {
      const float4 s = __ldcs(s4 + i);
      if (c.x > 0.0f) { acc += (double)s.x / (double)c.x; occ += 1.0; }
      if (c.y > 0.0f) { acc += (double)s.y / (double)c.y; occ += 1.0; }
      if (c.z > 0.0f) { acc += (double)s.z / (double)c.z; occ += 1.0; }
      if (c.w > 0.0f) { acc += (double)s.w / (double)c.w; occ += 1.0; }
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float c = grid[cells + i];
    if (c > 0.0f) { acc += (double)grid[i] / (double)c; occ += 1.0; }
  }
  acc = warp_sum(acc);
  occ = warp_sum(occ);
  __shared__ double sa[32], so[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sa[w] = acc; so[w] = occ; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, o = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { a += sa[q]; o += so[q]; }
    atomicAdd(out, a);
    atomicAdd(out + 1, o);
  }
}

// touched-voxel list: slots [0, n) (code or -1, duplicates allowed) then [n, n + *count) (appended).
// Each voxel is claimed once (atomicExch on its count), its sum / count accumulated and both
// entries zeroed: the grid is left clean.
__global__ void k_vox_mass_sparse(float* __restrict__ grid, int64_t cells, const int32_t* __restrict__ list,
                                  const int32_t* __restrict__ count, int64_t n, double* __restrict__ out) {
  const int64_t m = n + min((int64_t)*count, n);
  double acc = 0.0, occ = 0.0;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  // four list slots per thread and step: their claims (returning atomics) and sum reads are issued
  // back to back, so each thread waits on one memory round trip per 4 slots instead of per slot (the
  // loop is latency-bound). A voxel listed twice is claimed once: the second exchange returns 0.
  const bool vec = (reinterpret_cast<uintptr_t>(list) & 15u) == 0u;
  const int64_t m4 = vec ? m / 4 : 0;
  for (int64_t q = t0; q < m4; q += stride) {
    const int4 c4 = __ldg(reinterpret_cast<const int4*>(list) + q);
    const int32_t c[4] = {c4.x, c4.y, c4.z, c4.w};
    if ((c[0] & c[1] & c[2] & c[3]) < 0) continue;  // all four empty (-1)
    float cnt[4], rho[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cnt[k] = c[k] >= 0 ? atomicExch(grid + cells + c[k], 0.0f) : 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) rho[k] = cnt[k] > 0.0f ? grid[c[k]] : 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (cnt[k] > 0.0f) {
        acc += (double)rho[k] / (double)cnt[k];
        occ += 1.0;
        grid[c[k]] = 0.0f;
      }
  }
  for (int64_t j = 4 * m4 + t0; j < m; j += stride) {
    const int32_t c = __ldg(list + j);
    if (c < 0) continue;
    const float cnt = atomicExch(grid + cells + c, 0.0f);
    if (cnt > 0.0f) {
      acc += (double)grid[c] / (double)cnt;
      occ += 1.0;
      grid[c] = 0.0f;
    }
  }
  // block reduction first: one pair of fp64 atomics per block (same-address fp64 atomics serialise
  // in L2; one per warp cost ~0.1 ms at C5)
  __shared__ double s_acc[32], s_occ[32];
  acc = warp_sum(acc);
  occ = warp_sum(occ);
  const int wid = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  if ((threadIdx.x & 31) == 0) {
    s_acc[wid] = acc;
    s_occ[wid] = occ;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, o = 0.0;
    for (int q = 0; q < nw; ++q) {
      a += s_acc[q];
      o += s_occ[q];
    }
    if (a != 0.0 || o != 0.0) {
      atomicAdd(out, a);
      atomicAdd(out + 1, o);
    }
  }
}

__global__ void k_vox_scale(const double* __restrict__ lo_hi, int g, double* __restrict__ out) {
  double lo[3];
  const double e = voxel_edge(lo_hi, g, lo);
  out[0] = out[0] * (e * e * e);
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int pf_voxel_mass_sparse(float* grid, int32_t g, const int32_t* list, const int32_t* count, int64_t capacity,
                         const double* lo_hi, double* out, void* stream) {
  if (g < 1) return set_error(PF_ERR_VALUE, "voxel grid side must be >= 1");
  if (!list || !count) return set_error(PF_ERR_VALUE, "voxel_mass_sparse: list and count required");
  const int64_t cells = (int64_t)g * g * g;
  k_vox_mass_sparse<<<grid_for(2 * capacity, 256, 148 * 8), 256, 0, S(stream)>>>(grid, cells, list, count, capacity,
                                                                                  out);
  if (int rc = check_launch("voxel_mass_sparse")) return rc;
  k_vox_scale<<<1, 1, 0, S(stream)>>>(lo_hi, g, out);
  return check_launch("voxel_mass_scale");
}

int pf_bbox(const float* points, int64_t n, double* lo_hi, void* stream) {
  if (n <= 0) return set_error(PF_ERR_VALUE, "bbox of an empty point cloud");
  k_bbox_init<<<1, 32, 0, S(stream)>>>(reinterpret_cast<uint32_t*>(lo_hi));
  if (int rc = check_launch("bbox_init")) return rc;
  k_bbox_reduce<<<grid_for(n, 256, 148 * 4), 256, 0, S(stream)>>>(points, n,
                                                                  reinterpret_cast<uint32_t*>(lo_hi));
  if (int rc = check_launch("bbox_reduce")) return rc;
  k_bbox_final<<<1, 1, 0, S(stream)>>>(lo_hi);
  return check_launch("bbox_final");
}

int pf_voxel_codes(const float* points, int64_t n, const double* lo_hi, int32_t g, int32_t* codes,
                   void* stream) {
  if (g < 1 || g > 1290) return set_error(PF_ERR_VALUE, "voxel grid side must be in [1, 1290], got %d", g);
  if (n <= 0) return PF_OK;
  k_codes<<<grid_for(n, 256), 256, 0, S(stream)>>>(points, n, lo_hi, g, codes);
  return check_launch("voxel_codes");
}

int pf_voxel_accumulate(const int32_t* codes, const float* rho, int64_t n, int32_t g, float* grid,
                        void* stream) {
  if (g < 1 || g > 1290) return set_error(PF_ERR_VALUE, "voxel grid side must be in [1, 1290], got %d", g);
  if (n <= 0) return PF_OK;
  const int64_t cells = (int64_t)g * g * g;
  k_vox_acc<<<grid_for(n, 256), 256, 0, S(stream)>>>(codes, rho, n, cells, grid);
  return check_launch("voxel_accumulate");
}

int pf_voxel_mass(const float* grid, int32_t g, const double* lo_hi, double* out, void* stream) {
  if (g < 1 || g > 1290) return set_error(PF_ERR_VALUE, "voxel grid side must be in [1, 1290], got %d", g);
  const int64_t cells = (int64_t)g * g * g;
  k_vox_mass<<<grid_for(cells / 4 + 1, 256, 148 * 8), 256, 0, S(stream)>>>(grid, cells, out);
  if (int rc = check_launch("voxel_mass")) return rc;
  k_vox_scale<<<1, 1, 0, S(stream)>>>(lo_hi, g, out);
  return check_launch("voxel_mass_scale");
}

}  // extern "C"

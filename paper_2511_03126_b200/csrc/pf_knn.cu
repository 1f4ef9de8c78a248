// integrate.characteristic_length (integrate.py:72-95) on the device: the distance d_k from every
// point to its (k+1)-th nearest point, self included (cKDTree.query(p, k+1)[:, k]), and
// L = sqrt(pi / k * sum d_k^2).
//
// Uniform grid of cell c (1.25 x the expected k-NN spacing of a surface sample, from the bbox area),
// cells hashed into 2^22 buckets; points counting-sorted by bucket (cell id kept per point). A
// point's search starts with its 3 x 3 x 3 cell block and grows by shells until the (k+1)-th
// smallest squared distance found is inside the searched block (every unsearched point is then
// farther), so the result is exact. Distances in fp64 from the f32 coordinates, as the reference
// computes them on float64-upcast positions.
#include <cmath>

#include "pf_common.cuh"
#include "pf_tile.cuh"

namespace pf {
namespace {

constexpr int kHashLog = 22;
constexpr uint32_t kHashBins = 1u << kHashLog;
constexpr int kMaxK = 31;       // k + 1 <= 32 neighbours kept per point
constexpr int kCellBits = 11;   // cell coordinates < 2048 per axis

__device__ __forceinline__ uint32_t cell_hash(int cx, int cy, int cz) {
  return ((uint32_t)cx * 73856093u ^ (uint32_t)cy * 19349663u ^ (uint32_t)cz * 83492791u) & (kHashBins - 1);
}

struct Grid {
  float lo[3];
  float c;
  int dims[3];
};

__global__ void k_knn_grid(const double* __restrict__ lo_hi, int64_t n, int k, Grid* g) {
  // expected k-NN spacing of N points on a surface of area A: pi r^2 N / A = k + 1 -> r; A from the bbox
  const double ex = lo_hi[3] - lo_hi[0], ey = lo_hi[4] - lo_hi[1], ez = lo_hi[5] - lo_hi[2];
  const double area = fmax(2.0 * (ex * ey + ey * ez + ez * ex), 1e-30);
  double c = 1.25 * sqrt((double)(k + 1) * area / (3.141592653589793 * (double)n));
  const double ext = fmax(fmax(ex, ey), ez);
  c = fmax(c, ext / 2000.0);  // cell ids fit 11 bits per axis
  if (!(c > 0.0)) c = 1.0;
  g->c = (float)c;
  g->lo[0] = (float)lo_hi[0];
  g->lo[1] = (float)lo_hi[1];
  g->lo[2] = (float)lo_hi[2];
  g->dims[0] = (int)(ex / c) + 1;
  g->dims[1] = (int)(ey / c) + 1;
  g->dims[2] = (int)(ez / c) + 1;
}

__device__ __forceinline__ void cell_of(const Grid& g, float x, float y, float z, int& cx, int& cy, int& cz) {
  const float ic = 1.f / g.c;
  cx = min(max((int)((x - g.lo[0]) * ic), 0), g.dims[0] - 1);
  cy = min(max((int)((y - g.lo[1]) * ic), 0), g.dims[1] - 1);
  cz = min(max((int)((z - g.lo[2]) * ic), 0), g.dims[2] - 1);
}

__global__ void k_knn_keys(const float* __restrict__ p, int64_t n, const Grid* __restrict__ gp,
                           uint32_t* __restrict__ keys, uint32_t* __restrict__ hist) {
  const Grid g = *gp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int cx, cy, cz;
    cell_of(g, p[3 * i], p[3 * i + 1], p[3 * i + 2], cx, cy, cz);
    const uint32_t key = cell_hash(cx, cy, cz);
    keys[i] = key;
    atomicAdd(hist + key, 1u);
  }
}

__global__ void k_knn_scatter(const float* __restrict__ p, int64_t n, const Grid* __restrict__ gp,
                              const uint32_t* __restrict__ keys, uint32_t* __restrict__ cursor,
                              float4* __restrict__ kp, int32_t* __restrict__ kidx) {
  const Grid g = *gp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = p[3 * i], y = p[3 * i + 1], z = p[3 * i + 2];
    int cx, cy, cz;
    cell_of(g, x, y, z, cx, cy, cz);
    const uint32_t id = (uint32_t)cx | ((uint32_t)cy << kCellBits) | ((uint32_t)cz << (2 * kCellBits));
    const uint32_t pos = atomicAdd(cursor + keys[i], 1u);
    kp[pos] = make_float4(x, y, z, __uint_as_float(id));
    if (kidx) kidx[pos] = (int32_t)i;
  }
}

// one thread per point in bucket order (neighbouring threads query neighbouring cells). KP1 > 0:
// compile-time list length k + 1 (registers); KP1 == 0: runtime k (local memory)
template <int KP1>
__global__ void __launch_bounds__(128) k_knn_query(const float4* __restrict__ kp, int64_t n, const Grid* __restrict__ gp,
                                                   const uint32_t* __restrict__ ends, int k_rt, double* __restrict__ sum,
                                                   float* __restrict__ dk_sorted) {
  constexpr int kCap = KP1 > 0 ? KP1 : kMaxK + 1;
  const int k = KP1 > 0 ? KP1 - 1 : k_rt;
  const Grid g = *gp;
  const double c = (double)g.c;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 q = kp[i];
    const uint32_t id = __float_as_uint(q.w);
    const int cx = (int)(id & ((1u << kCellBits) - 1)), cy = (int)((id >> kCellBits) & ((1u << kCellBits) - 1)),
              cz = (int)(id >> (2 * kCellBits));
    const double qx = q.x, qy = q.y, qz = q.z;
    double best[kCap];
#pragma unroll
    for (int b = 0; b < kCap; ++b) best[b] = INFINITY;
    // distance from q to the faces of its own cell (the searched block of shell s reaches s*c beyond)
    const double fx = fmin(qx - ((double)g.lo[0] + cx * c), (double)g.lo[0] + (cx + 1) * c - qx);
    const double fy = fmin(qy - ((double)g.lo[1] + cy * c), (double)g.lo[1] + (cy + 1) * c - qy);
    const double fz = fmin(qz - ((double)g.lo[2] + cz * c), (double)g.lo[2] + (cz + 1) * c - qz);
    const double face = fmax(fmin(fmin(fx, fy), fz), 0.0);
    const int maxs = max(max(g.dims[0], g.dims[1]), g.dims[2]);
    for (int s = 1;; ++s) {
      for (int dz = -s; dz <= s; ++dz)
        for (int dy = -s; dy <= s; ++dy)
          for (int dx = -s; dx <= s; ++dx) {
            if (max(max(abs(dx), abs(dy)), abs(dz)) != s && s > 1) continue;  // shell only
            const int x = cx + dx, y = cy + dy, z = cz + dz;
            if (x < 0 || y < 0 || z < 0 || x >= g.dims[0] || y >= g.dims[1] || z >= g.dims[2]) continue;
            const uint32_t want = (uint32_t)x | ((uint32_t)y << kCellBits) | ((uint32_t)z << (2 * kCellBits));
            const uint32_t b = cell_hash(x, y, z);
            const uint32_t e0 = b ? __ldg(ends + b - 1) : 0u, e1 = __ldg(ends + b);
            for (uint32_t j = e0; j < e1; ++j) {
              const float4 r = __ldg(kp + j);
              if (__float_as_uint(r.w) != want) continue;
              const double ddx = (double)r.x - qx, ddy = (double)r.y - qy, ddz = (double)r.z - qz;
              double d2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
              if (d2 >= best[k]) continue;
              // insert into the ascending list best[0..k]
#pragma unroll
              for (int t = 0; t < kCap; ++t) {
                if (KP1 == 0 && t > k) break;
                const double lo = fmin(best[t], d2);
                d2 = fmax(best[t], d2);
                best[t] = lo;
              }
            }
          }
      // every unsearched point is at least face + (s - 1) * c + c away... block reaches face + s*c
      const double reach = face + (double)s * c;
      if (best[k] <= reach * reach || s >= maxs) break;
    }
    const double dk = sqrt(best[k]);
    if (dk_sorted) dk_sorted[i] = (float)dk;
    acc += best[k];
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, acc);
}

}  // namespace
}  // namespace pf

extern "C" {

uint64_t pf_knn_workspace_bytes(int64_t n) {
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  return al(sizeof(uint32_t) * (uint64_t)n) + al(sizeof(uint32_t) * pf::kHashBins) + al(sizeof(uint32_t) * 1024) +
         al(sizeof(float4) * (uint64_t)n) + al(sizeof(pf::Grid)) + al(6 * sizeof(double));
}

int pf_knn_kth_distance(const float* points, int64_t n, int32_t k, double* dk2_sum, float* dk_sorted,
                        void* workspace, void* stream) {
  using namespace pf;
  if (n < 1 || k < 0 || k > kMaxK || k >= n) return set_error(PF_ERR_VALUE, "knn: need 0 <= k < n and k <= %d", kMaxK);
  if (!workspace || !dk2_sum) return set_error(PF_ERR_VALUE, "knn: workspace and output required");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * (uint64_t)n);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * kHashBins);
  uint32_t* totals = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * 1024);
  float4* kp = reinterpret_cast<float4*>(ws);
  ws += al(sizeof(float4) * (uint64_t)n);
  Grid* g = reinterpret_cast<Grid*>(ws);
  ws += al(sizeof(Grid));
  double* lo_hi = reinterpret_cast<double*>(ws);
  if (int rc = pf_bbox(points, n, lo_hi, stream)) return rc;
  k_knn_grid<<<1, 1, 0, st>>>(lo_hi, n, k, g);
  if (int rc = check_launch("knn_grid")) return rc;
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kHashBins, st);
  cudaMemsetAsync(dk2_sum, 0, sizeof(double), st);
  k_knn_keys<<<grid_for(n, 256), 256, 0, st>>>(points, n, g, keys, hist);
  if (int rc = check_launch("knn_keys")) return rc;
  if (int rc = tile::run_bucket_scan(hist, totals, kHashBins, st)) return rc;
  k_knn_scatter<<<grid_for(n, 256), 256, 0, st>>>(points, n, g, keys, hist, kp, nullptr);
  if (int rc = check_launch("knn_scatter")) return rc;
  // after the scatter hist[b] = end of bucket b
  if (k == 8)  // AREA_KNN (integrate.py:19)
    k_knn_query<9><<<grid_for(n, 128, 148 * 32), 128, 0, st>>>(kp, n, g, hist, k, dk2_sum, dk_sorted);
  else
    k_knn_query<0><<<grid_for(n, 128, 148 * 32), 128, 0, st>>>(kp, n, g, hist, k, dk2_sum, dk_sorted);
  return check_launch("knn_query");
}

}  // extern "C"

// ---- geometry.estimate_normals (geometry.py:106-146) on the device -----------------------------------
// k nearest points (self included, cKDTree.query(p, k)) from the same exact grid search, their
// mean-centred covariance / k (numpy_impl.neighborhood_covariances), the eigenvector of the smallest
// eigenvalue (cyclic Jacobi in fp64, numpy.linalg.eigh order), the rank < 2 fallback to the camera
// direction and the orientation flip toward the mean camera centre.
namespace pf {
namespace {

__device__ void jacobi3(double a[3][3], double v[3][3], double w[3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 16; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double diag = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]);
    if (off <= 1e-300 || off <= 1e-18 * diag) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (a[p][q] == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J (columns p, q)
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- J^T A (rows p, q)
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {  // V <- V J
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  w[0] = a[0][0];
  w[1] = a[1][1];
  w[2] = a[2][2];
}

template <int K>
__global__ void __launch_bounds__(128) k_knn_normals(const float4* __restrict__ kp, const int32_t* __restrict__ kidx,
                                                     int64_t n, const Grid* __restrict__ gp,
                                                     const uint32_t* __restrict__ ends, double ccx, double ccy,
                                                     double ccz, double* __restrict__ normals,
                                                     uint8_t* __restrict__ degenerate) {
  const Grid g = *gp;
  const double c = (double)g.c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 q = kp[i];
    const uint32_t id = __float_as_uint(q.w);
    const int cx = (int)(id & ((1u << kCellBits) - 1)), cy = (int)((id >> kCellBits) & ((1u << kCellBits) - 1)),
              cz = (int)(id >> (2 * kCellBits));
    const double qx = q.x, qy = q.y, qz = q.z;
    double best[K];
    uint32_t bj[K];
#pragma unroll
    for (int b = 0; b < K; ++b) {
      best[b] = INFINITY;
      bj[b] = 0u;
    }
    const double fx = fmin(qx - ((double)g.lo[0] + cx * c), (double)g.lo[0] + (cx + 1) * c - qx);
    const double fy = fmin(qy - ((double)g.lo[1] + cy * c), (double)g.lo[1] + (cy + 1) * c - qy);
    const double fz = fmin(qz - ((double)g.lo[2] + cz * c), (double)g.lo[2] + (cz + 1) * c - qz);
    const double face = fmax(fmin(fmin(fx, fy), fz), 0.0);
    const int maxs = max(max(g.dims[0], g.dims[1]), g.dims[2]);
    for (int s = 1;; ++s) {
      for (int dz = -s; dz <= s; ++dz)
        for (int dy = -s; dy <= s; ++dy)
          for (int dx = -s; dx <= s; ++dx) {
            if (max(max(abs(dx), abs(dy)), abs(dz)) != s && s > 1) continue;
            const int x = cx + dx, y = cy + dy, z = cz + dz;
            if (x < 0 || y < 0 || z < 0 || x >= g.dims[0] || y >= g.dims[1] || z >= g.dims[2]) continue;
            const uint32_t want = (uint32_t)x | ((uint32_t)y << kCellBits) | ((uint32_t)z << (2 * kCellBits));
            const uint32_t b = cell_hash(x, y, z);
            const uint32_t e0 = b ? __ldg(ends + b - 1) : 0u, e1 = __ldg(ends + b);
            for (uint32_t j = e0; j < e1; ++j) {
              const float4 r = __ldg(kp + j);
              if (__float_as_uint(r.w) != want) continue;
              const double ddx = (double)r.x - qx, ddy = (double)r.y - qy, ddz = (double)r.z - qz;
              double d2 = fma(ddz, ddz, fma(ddy, ddy, ddx * ddx));
              if (d2 >= best[K - 1]) continue;
              uint32_t jj = j;
#pragma unroll
              for (int t = 0; t < K; ++t) {  // ascending insertion, index carried along
                const bool sw = d2 < best[t];
                const double lo = sw ? d2 : best[t], hi = sw ? best[t] : d2;
                const uint32_t jl = sw ? jj : bj[t], jh = sw ? bj[t] : jj;
                best[t] = lo;
                bj[t] = jl;
                d2 = hi;
                jj = jh;
              }
            }
          }
      const double reach = face + (double)s * c;
      if (best[K - 1] <= reach * reach || s >= maxs) break;
    }
    // neighbourhood covariance (numpy_impl.py:115-128): mean, centred outer products, / k
    double px[K], py[K], pz[K];
    double mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const float4 r = __ldg(kp + bj[t]);
      px[t] = r.x;
      py[t] = r.y;
      pz[t] = r.z;
      mx += px[t];
      my += py[t];
      mz += pz[t];
    }
    mx /= K;
    my /= K;
    mz /= K;
    double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const double d0 = px[t] - mx, d1 = py[t] - my, d2 = pz[t] - mz;
      a[0][0] += d0 * d0;
      a[0][1] += d0 * d1;
      a[0][2] += d0 * d2;
      a[1][1] += d1 * d1;
      a[1][2] += d1 * d2;
      a[2][2] += d2 * d2;
    }
    a[0][0] /= K; a[0][1] /= K; a[0][2] /= K; a[1][1] /= K; a[1][2] /= K; a[2][2] /= K;
    a[1][0] = a[0][1];
    a[2][0] = a[0][2];
    a[2][1] = a[1][2];
    double v[3][3], w[3];
    jacobi3(a, v, w);
    // ascending eigenvalues (eigh): the smallest one's vector, the middle and largest values
    int i0 = 0, i1 = 1, i2 = 2;
    if (w[i0] > w[i1]) { const int t = i0; i0 = i1; i1 = t; }
    if (w[i1] > w[i2]) { const int t = i1; i1 = i2; i2 = t; }
    if (w[i0] > w[i1]) { const int t = i0; i0 = i1; i1 = t; }
    double nx = v[0][i0], ny = v[1][i0], nz = v[2][i0];
    const double tx = ccx - qx, ty = ccy - qy, tz = ccz - qz;
    const bool degen = w[i1] <= 1e-10 * fmax(w[i2], 1e-300);  // geometry.py:13,136
    if (degen) {
      const double l = fmax(sqrt(tx * tx + ty * ty + tz * tz), 1e-30);
      nx = tx / l;
      ny = ty / l;
      nz = tz / l;
    }
    if (nx * tx + ny * ty + nz * tz < 0.0) {
      nx = -nx;
      ny = -ny;
      nz = -nz;
    }
    const double l = fmax(sqrt(nx * nx + ny * ny + nz * nz), 1e-30);
    const int64_t o = kidx[i];
    normals[3 * o] = nx / l;
    normals[3 * o + 1] = ny / l;
    normals[3 * o + 2] = nz / l;
    degenerate[o] = degen ? 1 : 0;
  }
}

}  // namespace
}  // namespace pf

extern "C" {

uint64_t pf_normals_workspace_bytes(int64_t n) {
  return pf_knn_workspace_bytes(n) + ((sizeof(int32_t) * (uint64_t)n + 255) & ~uint64_t(255));
}

int pf_estimate_normals(const float* points, int64_t n, int32_t k, double ccx, double ccy, double ccz,
                        double* normals, uint8_t* degenerate, void* workspace, void* stream) {
  using namespace pf;
  if (k < 3) return set_error(PF_ERR_VALUE, "normal estimation needs k >= 3, got %d", k);
  if (k > n) return set_error(PF_ERR_VALUE, "k=%d exceeds point count %lld", k, (long long)n);
  if (k != 16 && k != 8 && k != 3 && k != 4 && k != 6 && k != 10 && k != 12 && k != 20 && k != 24 && k != 32)
    return set_error(PF_ERR_VALUE, "estimate_normals: k=%d not compiled (3, 4, 6, 8, 10, 12, 16, 20, 24, 32)", k);
  if (!workspace || !normals || !degenerate) return set_error(PF_ERR_VALUE, "estimate_normals: null buffer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * (uint64_t)n);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * kHashBins);
  uint32_t* totals = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * 1024);
  float4* kp = reinterpret_cast<float4*>(ws);
  ws += al(sizeof(float4) * (uint64_t)n);
  Grid* g = reinterpret_cast<Grid*>(ws);
  ws += al(sizeof(Grid));
  double* lo_hi = reinterpret_cast<double*>(ws);
  ws += al(6 * sizeof(double));
  int32_t* kidx = reinterpret_cast<int32_t*>(ws);
  if (int rc = pf_bbox(points, n, lo_hi, stream)) return rc;
  k_knn_grid<<<1, 1, 0, st>>>(lo_hi, n, k - 1, g);
  if (int rc = check_launch("normals_grid")) return rc;
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kHashBins, st);
  k_knn_keys<<<grid_for(n, 256), 256, 0, st>>>(points, n, g, keys, hist);
  if (int rc = check_launch("normals_keys")) return rc;
  if (int rc = tile::run_bucket_scan(hist, totals, kHashBins, st)) return rc;
  k_knn_scatter<<<grid_for(n, 256), 256, 0, st>>>(points, n, g, keys, hist, kp, kidx);
  if (int rc = check_launch("normals_scatter")) return rc;
  const int blocks = grid_for(n, 128, 148 * 32);
#define PF_NORMALS_K(KK) \
  case KK: k_knn_normals<KK><<<blocks, 128, 0, st>>>(kp, kidx, n, g, hist, ccx, ccy, ccz, normals, degenerate); break;
  switch (k) {
    PF_NORMALS_K(3) PF_NORMALS_K(4) PF_NORMALS_K(6) PF_NORMALS_K(8) PF_NORMALS_K(10) PF_NORMALS_K(12)
    PF_NORMALS_K(16) PF_NORMALS_K(20) PF_NORMALS_K(24) PF_NORMALS_K(32)
  }
#undef PF_NORMALS_K
  return check_launch("normals_query");
}

}  // extern "C"

// ---- nearest point of another set (densify_field's donor query, densify.py:142-147) --------------------
// Grid over the donor points (the k-NN grid above with k = 1), each query searches shells around its
// cell until its best fp64 squared distance is inside the searched block; lowest donor index on ties
// (as a brute-force scan would give).
namespace pf {
namespace {

__device__ __forceinline__ unsigned long long dflip(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(d);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunflip(unsigned long long u) {
  u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
  return __longlong_as_double((long long)u);
}

__global__ void k_bbox64(const double* __restrict__ p, int64_t n, unsigned long long* __restrict__ mm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int a = 0; a < 3; ++a) {
      const unsigned long long f = dflip(p[3 * i + a]);
      atomicMin(mm + a, f);
      atomicMax(mm + 3 + a, f);
    }
}

__global__ void k_bbox64_final(const unsigned long long* __restrict__ mm, double* __restrict__ lo_hi) {
  if (threadIdx.x < 6) lo_hi[threadIdx.x] = dunflip(mm[threadIdx.x]);
}

__global__ void k_f64_to_f32(const double* __restrict__ p, int64_t n3, float* __restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n3; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = (float)p[i];
}

__global__ void __launch_bounds__(128) k_cross_nearest(const double* __restrict__ qp, int64_t nq,
                                                       const double* __restrict__ pp, int64_t np,
                                                       const float4* __restrict__ kp,
                                                       const int32_t* __restrict__ kidx, const Grid* __restrict__ gp,
                                                       const uint32_t* __restrict__ ends, int64_t* __restrict__ out) {
  const Grid g = *gp;
  const double c = (double)g.c;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    const double qx = qp[3 * i], qy = qp[3 * i + 1], qz = qp[3 * i + 2];
    double bd = INFINITY;
    int64_t bi = INT64_MAX;
    const double gx1 = (double)g.lo[0] + g.dims[0] * c, gy1 = (double)g.lo[1] + g.dims[1] * c,
                 gz1 = (double)g.lo[2] + g.dims[2] * c;
    if (!(qx >= g.lo[0] && qx < gx1 && qy >= g.lo[1] && qy < gy1 && qz >= g.lo[2] && qz < gz1)) {
      // outside the donors' grid (rare): the shell bound does not apply, scan every donor
      for (int64_t o = 0; o < np; ++o) {
        const double ex = __dsub_rn(qx, pp[3 * o]), ey = __dsub_rn(qy, pp[3 * o + 1]), ez = __dsub_rn(qz, pp[3 * o + 2]);
        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
        if (d2 < bd) {  // ascending o: the first minimum is the lowest index
          bd = d2;
          bi = o;
        }
      }
      out[i] = bi;
      continue;
    }
    int cx, cy, cz;
    cell_of(g, (float)qx, (float)qy, (float)qz, cx, cy, cz);
    const int maxs = max(max(g.dims[0], g.dims[1]), g.dims[2]);
    for (int s = 0;; ++s) {
      // shell s (cells at Chebyshev distance s), clipped to the grid: O(s^2) cells per shell
      const int z0 = max(cz - s, 0), z1 = min(cz + s, g.dims[2] - 1);
      const int y0 = max(cy - s, 0), y1 = min(cy + s, g.dims[1] - 1);
      for (int z = z0; z <= z1; ++z)
        for (int y = y0; y <= y1; ++y) {
          const bool face = abs(z - cz) == s || abs(y - cy) == s;
          const int xs = face ? 1 : 2 * s;  // interior rows of the cube: only x = cx -+ s
          for (int x = cx - s; x <= cx + s; x += (s == 0 ? 1 : xs)) {
            if (x < 0 || x >= g.dims[0]) continue;
            const uint32_t want = (uint32_t)x | ((uint32_t)y << kCellBits) | ((uint32_t)z << (2 * kCellBits));
            const uint32_t b = cell_hash(x, y, z);
            const uint32_t e0 = b ? __ldg(ends + b - 1) : 0u, e1 = __ldg(ends + b);
            for (uint32_t j = e0; j < e1; ++j) {
              if (__float_as_uint(__ldg(&kp[j].w)) != want) continue;
              const int64_t o = __ldg(kidx + j);
              const double ex = __dsub_rn(qx, pp[3 * o]), ey = __dsub_rn(qy, pp[3 * o + 1]),
                           ez = __dsub_rn(qz, pp[3 * o + 2]);
              const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez));
              if (d2 < bd || (d2 == bd && o < bi)) {
                bd = d2;
                bi = o;
              }
            }
          }
        }
      // every donor outside the searched block [c - s, c + s] is at least `reach` away from q
      const double bx0 = (double)g.lo[0] + (cx - s) * c, bx1 = (double)g.lo[0] + (cx + s + 1) * c;
      const double by0 = (double)g.lo[1] + (cy - s) * c, by1 = (double)g.lo[1] + (cy + s + 1) * c;
      const double bz0 = (double)g.lo[2] + (cz - s) * c, bz1 = (double)g.lo[2] + (cz + s + 1) * c;
      const double reach = fmax(fmin(fmin(fmin(qx - bx0, bx1 - qx), fmin(qy - by0, by1 - qy)),
                                     fmin(qz - bz0, bz1 - qz)), 0.0) * (1.0 - 1e-9);
      if ((bi != INT64_MAX && bd < reach * reach) || s >= maxs) break;
    }
    out[i] = bi;
  }
}

}  // namespace
}  // namespace pf

extern "C" {

uint64_t pf_nearest_workspace_bytes(int64_t np) {
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  return pf_knn_workspace_bytes(np) + al(sizeof(int32_t) * (uint64_t)np) + al(sizeof(float) * 3 * (uint64_t)np) +
         al(8 * sizeof(unsigned long long));
}

int pf_nearest_index_grid(const double* queries, int64_t nq, const double* points, int64_t np, int64_t* idx,
                          void* workspace, void* stream) {
  using namespace pf;
  if (nq < 0 || np < 0) return set_error(PF_ERR_VALUE, "nearest_index: negative size");
  if (nq == 0) return PF_OK;
  if (np == 0) return set_error(PF_ERR_MATERIAL, "no point in the cloud has a geometric feature");
  if (!workspace) return set_error(PF_ERR_VALUE, "nearest_index: workspace missing");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  uint32_t* keys = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * (uint64_t)np);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * kHashBins);
  uint32_t* totals = reinterpret_cast<uint32_t*>(ws);
  ws += al(sizeof(uint32_t) * 1024);
  float4* kp = reinterpret_cast<float4*>(ws);
  ws += al(sizeof(float4) * (uint64_t)np);
  Grid* g = reinterpret_cast<Grid*>(ws);
  ws += al(sizeof(Grid));
  double* lo_hi = reinterpret_cast<double*>(ws);
  ws += al(6 * sizeof(double));
  int32_t* kidx = reinterpret_cast<int32_t*>(ws);
  ws += al(sizeof(int32_t) * (uint64_t)np);
  float* p32 = reinterpret_cast<float*>(ws);
  ws += al(sizeof(float) * 3 * (uint64_t)np);
  unsigned long long* mm = reinterpret_cast<unsigned long long*>(ws);
  cudaMemsetAsync(mm, 0xff, 3 * sizeof(unsigned long long), st);
  cudaMemsetAsync(mm + 3, 0, 3 * sizeof(unsigned long long), st);
  k_bbox64<<<grid_for(np, 256), 256, 0, st>>>(points, np, mm);
  k_bbox64_final<<<1, 32, 0, st>>>(mm, lo_hi);
  k_f64_to_f32<<<grid_for(3 * np, 256), 256, 0, st>>>(points, 3 * np, p32);
  if (int rc = check_launch("nearest_bbox")) return rc;
  k_knn_grid<<<1, 1, 0, st>>>(lo_hi, np, 1, g);
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kHashBins, st);
  k_knn_keys<<<grid_for(np, 256), 256, 0, st>>>(p32, np, g, keys, hist);
  if (int rc = check_launch("nearest_keys")) return rc;
  if (int rc = tile::run_bucket_scan(hist, totals, kHashBins, st)) return rc;
  k_knn_scatter<<<grid_for(np, 256), 256, 0, st>>>(p32, np, g, keys, hist, kp, kidx);
  if (int rc = check_launch("nearest_scatter")) return rc;
  k_cross_nearest<<<grid_for(nq, 128, 148 * 32), 128, 0, st>>>(queries, nq, points, np, kp, kidx, g, hist, idx);
  return check_launch("nearest_query");
}

}  // extern "C"

// ---- integrate_mass partials from a probability matrix (integrate.py:124-155) -------------------------
namespace pf {
namespace {
constexpr int kIntWarps = 8;
__global__ void __launch_bounds__(32 * kIntWarps) k_integrate_partials(const double* __restrict__ w, int64_t n, int k,
                                                                         const float* __restrict__ pos,
                                                                         const float* __restrict__ nrm,
                                                                         const double* __restrict__ mt,
                                                                         const double* __restrict__ th,
                                                                         double* __restrict__ out) {
  __shared__ double red[kIntWarps][4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double wt[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // weight totals of columns lane + 32 j
  double pm_s = 0.0, px = 0.0, py = 0.0, pz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kIntWarps + wid; i < n; i += (int64_t)gridDim.x * kIntWarps) {
    const double* row = w + i * k;
    double pm = 0.0, mth = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kk = lane + 32 * j;
      if (kk < k) {
        const double v = row[kk];
        wt[j] += v;
        pm = fma(v, mt[kk], pm);
        mth = fma(v, th[kk], mth);
      }
    }
    pm = warp_sum(pm);
    mth = warp_sum(mth);
    double cx = pos[3 * i], cy = pos[3 * i + 1], cz = pos[3 * i + 2];
    if (nrm) {
      const double h = mth / 2.0;
      cx -= h * nrm[3 * i];
      cy -= h * nrm[3 * i + 1];
      cz -= h * nrm[3 * i + 2];
    }
    pm_s += pm;
    px += pm * cx;
    py += pm * cy;
    pz += pm * cz;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (lane + 32 * j < k && wt[j] != 0.0) atomicAdd(out + lane + 32 * j, wt[j]);
  if (lane == 0) {
    red[wid][0] = pm_s;
    red[wid][1] = px;
    red[wid][2] = py;
    red[wid][3] = pz;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double s = 0.0;
    for (int q = 0; q < kIntWarps; ++q) s += red[q][threadIdx.x];
    if (s != 0.0) atomicAdd(out + k + threadIdx.x, s);
  }
}
}  // namespace
}  // namespace pf

extern "C" int pf_integrate_partials(const double* weights, int64_t n, int32_t k, const float* positions,
                                     const float* normals, const double* mid_theta, const double* theta,
                                     double* out, void* stream) {
  using namespace pf;
  if (n < 0 || k < 1 || k > 256) return set_error(PF_ERR_VALUE, "integrate_partials: need 1 <= k <= 256");
  if (n == 0) return PF_OK;
  k_integrate_partials<<<grid_for(n, kIntWarps, 148 * 8), 32 * kIntWarps, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      weights, n, k, positions, normals, mid_theta, theta, out);
  return check_launch("integrate_partials");
}

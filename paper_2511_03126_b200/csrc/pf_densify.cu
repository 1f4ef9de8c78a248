// Densification: `dino_knn_interpolate` (densify.py:36-86) and the orphan step of
// `densify_field` (densify.py:110-160) on the device, fp64 like the reference.
//
// dino_knn_interpolate(q (Q,D), s (S,D), probs (S,M), k):
//   qn = q / |q| (zero rows -> MaterialError listing them), su = s / max(|s|, 1e-30),
//   sims = qn @ su^T                                    k_dk_sims: 64x64-tiled fp64 SIMT GEMM
//   neighbours = the k best by (-sim, index)            k_dk_select: warp per query, k rounds of
//                                                       "best key strictly after the previous pick"
//                                                       (no taken-mask: picks come out in order)
//   w = max(sim, 0) / sum (uniform 1/k when the sum is <= 0); out = sum_j w_j probs[n_j]
// The neighbour order and tie-break are the reference's (descending similarity, lower index first,
// densify.py:69-74); k == S gives the full stable argsort. Sums run in the reference's order
// (left to right over the neighbours), so results agree with numpy to BLAS rounding (1e-12).
//
// nearest_index(queries (A,3), points (B,3)): brute-force exact nearest point in fp64 with lowest
// index on ties — the cKDTree(k=1) query that gives featureless points their donor (densify.py:
// 142-147); the orphan set is small (points visible in no view).
#include <cfloat>
#include <cstdio>
#include <vector>

#include "pf_common.cuh"

namespace pf {
namespace {

constexpr int kT = 64;        // GEMM tile (queries x sources)
constexpr int kKc = 16;       // depth chunk
constexpr int kSelWarps = 4;  // select kernel warps per block
constexpr int kMaxK = 1024;

__global__ void k_dk_rownorm(const double* __restrict__ x, int64_t rows, int d, double* __restrict__ norm,
                             uint8_t* __restrict__ zero, int32_t* __restrict__ nzero) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < rows; r += nw) {
    double acc = 0.0;
    for (int c = lane; c < d; c += 32) {
      const double v = x[r * d + c];
      acc = fma(v, v, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) {
      const double nr = sqrt(acc);
      norm[r] = nr;
      if (zero) {
        const bool z = nr == 0.0;
        zero[r] = z ? 1 : 0;
        if (z) atomicAdd(nzero, 1);
      }
    }
  }
}

// sims[i, j] = sum_c (q[i,c] / qn[i]) * (s[j,c] / max(sn[j], 1e-30))
__global__ void __launch_bounds__(256) k_dk_sims(const double* __restrict__ q, const double* __restrict__ qn,
                                                 int64_t nq, const double* __restrict__ s,
                                                 const double* __restrict__ sn, int64_t ns, int d,
                                                 double* __restrict__ sims) {
  __shared__ double A[kKc][kT + 1], B[kKc][kT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = (int64_t)blockIdx.y * kT, j0 = (int64_t)blockIdx.x * kT;
  double acc[4][4] = {};
  for (int c0 = 0; c0 < d; c0 += kKc) {
    for (int e = threadIdx.x; e < kKc * kT; e += 256) {
      const int r = e / kKc, c = e % kKc;
      const int64_t qi = i0 + r, sj = j0 + r;
      double a = 0.0, b = 0.0;
      if (qi < nq && c0 + c < d) a = __ddiv_rn(q[qi * d + c0 + c], qn[qi]);
      if (sj < ns && c0 + c < d) b = __ddiv_rn(s[sj * d + c0 + c], fmax(sn[sj], 1e-30));
      A[c][r] = a;
      B[c][r] = b;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < kKc; ++c) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = A[c][ty + 16 * u];
        b[u] = B[c][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t qi = i0 + ty + 16 * u, sj = j0 + tx + 16 * v;
      if (qi < nq && sj < ns) sims[qi * ns + sj] = acc[u][v];
    }
}

// a before b in the reference's neighbour order: higher similarity, then lower index
__device__ __forceinline__ bool before(double sa, int64_t ia, double sb, int64_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

__global__ void __launch_bounds__(kSelWarps * 32) k_dk_select(const double* __restrict__ sims, int64_t nq,
                                                              int64_t ns, int k, const double* __restrict__ probs,
                                                              int m, double* __restrict__ out,
                                                              int32_t* __restrict__ nbr_out) {
  extern __shared__ unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* s_sim = reinterpret_cast<double*>(smem) + (size_t)warp * k;
  int32_t* s_idx = reinterpret_cast<int32_t*>(reinterpret_cast<double*>(smem) + (size_t)kSelWarps * k) +
                   (size_t)warp * k;
  for (int64_t qi = blockIdx.x * (int64_t)kSelWarps + warp; qi < nq; qi += (int64_t)gridDim.x * kSelWarps) {
    const double* row = sims + qi * ns;
    double prev_s = DBL_MAX;  // sentinel before every real key
    int64_t prev_i = -1;
    for (int r = 0; r < k; ++r) {
      double bs = -DBL_MAX;
      int64_t bi = INT64_MAX;
      for (int64_t j = lane; j < ns; j += 32) {
        const double sj = row[j];
        if (before(prev_s, prev_i, sj, j) && before(sj, j, bs, bi)) {
          bs = sj;
          bi = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (before(os, oi, bs, bi)) {
          bs = os;
          bi = oi;
        }
      }
      if (lane == 0) {  // NaN similarities are never picked: their slots poison the row with NaN
        s_sim[r] = bi < ns ? bs : __longlong_as_double(0x7ff8000000000000ll);
        s_idx[r] = bi < ns ? (int32_t)bi : 0;
      }
      prev_s = bs;
      prev_i = bi;
    }
    __syncwarp();
    // weights: clamp at zero, normalise; uniform when every clamped weight vanishes (densify.py:77-83)
    double total = 0.0;
    for (int r = 0; r < k; ++r) total += fmax(s_sim[r], 0.0);
    const bool flat = total <= 0.0;
    if (flat) total = (double)k;
    for (int c = lane; c < m; c += 32) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r) {
        const double w = __ddiv_rn(flat ? 1.0 : fmax(s_sim[r], 0.0), total);
        acc = __fma_rn(w, probs[(int64_t)s_idx[r] * m + c], acc);
      }
      out[qi * m + c] = acc;
    }
    if (nbr_out)
      for (int r = lane; r < k; r += 32) nbr_out[qi * k + r] = s_idx[r];
    __syncwarp();
  }
}

// nearest point (fp64 squared distance, lowest index on ties), one warp per query
__global__ void k_nearest(const double* __restrict__ qp, int64_t nq, const double* __restrict__ pp, int64_t np,
                          int64_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < nq; i += nw) {
    const double x = qp[3 * i], y = qp[3 * i + 1], z = qp[3 * i + 2];
    double bd = DBL_MAX;
    int64_t bi = INT64_MAX;
    for (int64_t j = lane; j < np; j += 32) {
      const double dx = __dsub_rn(x, pp[3 * j]), dy = __dsub_rn(y, pp[3 * j + 1]), dz = __dsub_rn(z, pp[3 * j + 2]);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      if (d2 < bd) {  // j increases per lane: the first hit keeps the lowest index
        bd = d2;
        bi = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (od < bd || (od == bd && oi < bi)) {
        bd = od;
        bi = oi;
      }
    }
    if (lane == 0) idx[i] = bi;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

uint64_t pf_dino_knn_workspace_bytes(int64_t nq, int64_t ns, int32_t d) {
  (void)d;
  if (nq < 0 || ns < 0) return 0;
  return a256(sizeof(double) * nq) + a256(sizeof(double) * ns) + a256(sizeof(double) * nq * ns) + a256(nq) +
         a256(sizeof(int32_t));
}

int pf_dino_knn_interpolate(const double* q, int64_t nq, const double* s, int64_t ns, int32_t d,
                            const double* probs, int32_t m, int32_t k, double* out, int32_t* neighbors,
                            void* workspace, void* stream) {
  if (k < 1 || k > ns) return set_error(PF_ERR_VALUE, "k=%d outside 1..%lld", k, (long long)ns);
  if (k > kMaxK) return set_error(PF_ERR_VALUE, "k=%d above the supported %d", k, kMaxK);
  if (d < 1 || m < 1 || nq < 0) return set_error(PF_ERR_STRUCTURE, "dino_knn: bad shapes d=%d m=%d", d, m);
  if (nq == 0) return PF_OK;
  if (!q || !s || !probs || !out || !workspace) return set_error(PF_ERR_VALUE, "dino_knn: null buffer");
  unsigned char* w = reinterpret_cast<unsigned char*>(workspace);
  double* qn = reinterpret_cast<double*>(w);
  w += a256(sizeof(double) * nq);
  double* sn = reinterpret_cast<double*>(w);
  w += a256(sizeof(double) * ns);
  double* sims = reinterpret_cast<double*>(w);
  w += a256(sizeof(double) * nq * ns);
  uint8_t* zero = w;
  w += a256(nq);
  int32_t* nzero = reinterpret_cast<int32_t*>(w);
  cudaStream_t st = S(stream);
  cudaMemsetAsync(nzero, 0, sizeof(int32_t), st);
  k_dk_rownorm<<<grid_for(nq * 32, 256), 256, 0, st>>>(q, nq, d, qn, zero, nzero);
  if (int rc = check_launch("dino_knn_qnorm")) return rc;
  k_dk_rownorm<<<grid_for(ns * 32, 256), 256, 0, st>>>(s, ns, d, sn, nullptr, nullptr);
  if (int rc = check_launch("dino_knn_snorm")) return rc;
  // zero-norm queries raise MaterialError with their indices (densify.py:62-64): one host sync
  int32_t h_nzero = 0;
  cudaMemcpyAsync(&h_nzero, nzero, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("dino_knn_sync");
  if (h_nzero > 0) {
    std::vector<uint8_t> flags(nq);
    cudaMemcpy(flags.data(), zero, nq, cudaMemcpyDeviceToHost);
    char buf[256];
    int len = snprintf(buf, sizeof(buf), "query features missing for indices [");
    int listed = 0;
    for (int64_t i = 0; i < nq && listed < 10; ++i)
      if (flags[i]) len += snprintf(buf + len, sizeof(buf) - len, "%s%lld", listed++ ? ", " : "", (long long)i);
    snprintf(buf + len, sizeof(buf) - len, "]");
    return set_error(PF_ERR_MATERIAL, "%s", buf);
  }
  dim3 g((unsigned)((ns + kT - 1) / kT), (unsigned)((nq + kT - 1) / kT));
  if (g.y > 65535u) return set_error(PF_ERR_VALUE, "dino_knn: too many queries per call (%lld)", (long long)nq);
  k_dk_sims<<<g, 256, 0, st>>>(q, qn, nq, s, sn, ns, d, sims);
  if (int rc = check_launch("dino_knn_sims")) return rc;
  const size_t smem = (sizeof(double) + sizeof(int32_t)) * kSelWarps * (size_t)k;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_dk_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_dk_select<<<grid_for(nq, kSelWarps, 148 * 16), kSelWarps * 32, smem, st>>>(sims, nq, ns, k, probs, m, out,
                                                                                neighbors);
  return check_launch("dino_knn_select");
}

int pf_nearest_index(const double* queries, int64_t nq, const double* points, int64_t np, int64_t* idx,
                     void* stream) {
  if (nq < 0 || np < 0) return set_error(PF_ERR_VALUE, "nearest_index: negative size");
  if (nq == 0) return PF_OK;
  if (np == 0) return set_error(PF_ERR_MATERIAL, "no point in the cloud has a geometric feature");
  k_nearest<<<grid_for(nq * 32, 256), 256, 0, S(stream)>>>(queries, nq, points, np, idx);
  return check_launch("nearest_index");
}

}  // extern "C"

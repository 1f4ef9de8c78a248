// View scoring for the anchor set: view_select.score_views / rank_views
// (view_select.py:51-124) for all (anchor, view) pairs at once, fp64 in the reference's expressions.
//   pixels, z = project_points (numpy order, pf_common.cuh project); centre = -R^T t;
//   v_dir = (p - centre) / max(|p - centre|, 1e-30); s_angle = max(0, v_dir . -n);
//   s_dist = 1 / (1 + z); s_total = visible & z > 0 ? s_dist * s_angle : 0;
//   ranked: per anchor the k best visible views by (-s_total, view index), -1 padded.
// One warp per anchor: lanes over views, then k rounds of a warp argmax.
#include <cfloat>

#include "pf_common.cuh"

namespace pf {
namespace {

__global__ void k_score_views(const double* __restrict__ pos, const double* __restrict__ nrm, int64_t s,
                              const pf_view_t* __restrict__ views, int nv, const uint8_t* __restrict__ vis,
                              double* __restrict__ s_total, double* __restrict__ s_angle, double* __restrict__ zout,
                              double* __restrict__ pix, int k, int32_t* __restrict__ ranked) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < s; i += nw) {
    const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
    const double nx = nrm[3 * i], ny = nrm[3 * i + 1], nz = nrm[3 * i + 2];
    for (int j = lane; j < nv; j += 32) {
      const pf_view_t& v = views[j];
      const Proj q = project(v, px, py, pz);
      // centre = -R^T t (bundle.py:58-60)
      const double c0 = -fma(v.R[6], v.t[2], fma(v.R[3], v.t[1], v.R[0] * v.t[0]));
      const double c1 = -fma(v.R[7], v.t[2], fma(v.R[4], v.t[1], v.R[1] * v.t[0]));
      const double c2 = -fma(v.R[8], v.t[2], fma(v.R[5], v.t[1], v.R[2] * v.t[0]));
      const double tx = px - c0, ty = py - c1, tz = pz - c2;
      const double dist = fmax(sqrt(tx * tx + ty * ty + tz * tz), 1e-30);
      const double vx = tx / dist, vy = ty / dist, vz = tz / dist;
      const double sa = fmax(0.0, vx * -nx + vy * -ny + vz * -nz);
      const double sd = 1.0 / (1.0 + q.z);
      const bool ok = vis[i * nv + j] != 0 && q.z > 0.0;
      const int64_t o = i * nv + j;
      s_total[o] = ok ? sd * sa : 0.0;
      s_angle[o] = sa;
      zout[o] = q.z;
      pix[2 * o] = q.u;
      pix[2 * o + 1] = q.v;
    }
    __syncwarp();
    // k best visible views, (-s_total, index) order
    double prev_s = DBL_MAX;
    int prev_j = -1;
    for (int r = 0; r < k; ++r) {
      double bs = -DBL_MAX;
      int bj = INT32_MAX;
      for (int j = lane; j < nv; j += 32) {
        const int64_t o = i * nv + j;
        if (!(vis[o] != 0 && zout[o] > 0.0)) continue;
        const double sj = s_total[o];
        const bool after = sj < prev_s || (sj == prev_s && j > prev_j);
        const bool better = sj > bs || (sj == bs && j < bj);
        if (after && better) {
          bs = sj;
          bj = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, bs, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (os > bs || (os == bs && oj < bj)) {
          bs = os;
          bj = oj;
        }
      }
      if (lane == 0) ranked[i * k + r] = bj == INT32_MAX ? -1 : bj;
      if (bj == INT32_MAX) {
        for (int rr = r + 1 + lane; rr < k; rr += 32) ranked[i * k + rr] = -1;
        break;
      }
      prev_s = bs;
      prev_j = bj;
    }
  }
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_score_views(const double* positions, const double* normals, int64_t s, const pf_view_t* views,
                              int32_t nviews, const uint8_t* visibility, double* s_total, double* s_angle, double* z,
                              double* pixels, int32_t k, int32_t* ranked, void* stream) {
  if (k < 1) return set_error(PF_ERR_VALUE, "k must be >= 1, got %d", k);
  if (s < 0 || nviews < 1) return set_error(PF_ERR_STRUCTURE, "score_views: bad shapes");
  if (s == 0) return PF_OK;
  k_score_views<<<grid_for(s * 32, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      positions, normals, s, views, nviews, visibility, s_total, s_angle, z, pixels, k, ranked);
  return check_launch("score_views");
}

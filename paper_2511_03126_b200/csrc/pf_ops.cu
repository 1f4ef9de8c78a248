// Operator- and function-level kernels of the drop-in API, fp64, bit-exact with the reference.
//
// These back the reference's own plugin/operator surface — the `propfield.kernels` registry
// (kernels/__init__.py:21-101) and the geometry / fusion / grounding entry points that
// pipeline.py:224-232,275-281 calls — so existing callers and tests run unchanged on the GPU.
// They keep the reference's fp64 arithmetic and operation order (no FMA contraction) and therefore
// agree with numpy to the last bit; the throughput path is pf_fused.cu.
#include "pf_common.cuh"

namespace pf {
namespace {

// ---- kernels.visible_in_view (numpy_impl.py:14-40) ------------------------------------------------
__global__ void k_visible_in_view(const double* __restrict__ u, const double* __restrict__ v,
                                  const double* __restrict__ z, int64_t n,
                                  const float* __restrict__ depth, int h, int w, double eps,
                                  uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = depth_test(depth, h, w, u[i], v[i], z[i], eps) ? 1 : 0;
}

// one bilinear sample in the reference's fp64 operation order (numpy_impl.py:58-66)
template <int DT>
__device__ __forceinline__ double bilinear_sample(const void* fmap, const Taps& t, int wf, int d,
                                                  int c) {
  const double w00 = __dmul_rn(__dsub_rn(1.0, t.wy), __dsub_rn(1.0, t.wx));
  const double w01 = __dmul_rn(__dsub_rn(1.0, t.wy), t.wx);
  const double w10 = __dmul_rn(t.wy, __dsub_rn(1.0, t.wx));
  const double w11 = __dmul_rn(t.wy, t.wx);
  const double f00 = load_feat<DT>(fmap, ((int64_t)t.y0 * wf + t.x0) * d + c);
  const double f01 = load_feat<DT>(fmap, ((int64_t)t.y0 * wf + t.x1) * d + c);
  const double f10 = load_feat<DT>(fmap, ((int64_t)t.y1 * wf + t.x0) * d + c);
  const double f11 = load_feat<DT>(fmap, ((int64_t)t.y1 * wf + t.x1) * d + c);
  double acc = __dadd_rn(__dmul_rn(f00, w00), __dmul_rn(f01, w01));
  acc = __dadd_rn(acc, __dmul_rn(f10, w10));
  return __dadd_rn(acc, __dmul_rn(f11, w11));
}

// ---- kernels.bilinear_gather / accumulate_features (numpy_impl.py:43-77) ---------------------------
// warp per sample row, lanes over channels (coalesced along the channel-last map)
template <int DT, bool ACCUM>
__global__ void k_gather(const void* __restrict__ fmap, int hf, int wf, int d,
                         const double* __restrict__ fu, const double* __restrict__ fv, int64_t m,
                         const int64_t* __restrict__ rows, double* __restrict__ out,
                         int64_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m;
       i += warps) {
    const Taps t = make_taps(fu[i], fv[i], hf, wf);
    const int64_t r = ACCUM ? rows[i] : i;
    double* dst = out + r * d;
    for (int c = lane; c < d; c += 32) {
      const double s = bilinear_sample<DT>(fmap, t, wf, d, c);
      dst[c] = ACCUM ? __dadd_rn(dst[c], s) : s;
    }
    if (ACCUM && lane == 0) counts[r] += 1;
  }
}

// ---- geometry.project_points (geometry.py:46-59) ------------------------------------------------
__global__ void k_project(const double* __restrict__ p, int64_t n, pf_view_t vw,
                          double* __restrict__ uv, double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Proj q = project(vw, p[3 * i], p[3 * i + 1], p[3 * i + 2]);
    uv[2 * i] = q.u;
    uv[2 * i + 1] = q.v;
    z[i] = q.z;
  }
}

template <int PT>
__device__ __forceinline__ void load_point(const void* pts, int64_t i, double& x, double& y,
                                           double& z) {
  if constexpr (PT == PF_F64) {
    const double* p = reinterpret_cast<const double*>(pts) + 3 * i;
    x = p[0]; y = p[1]; z = p[2];
  } else {
    const float* p = reinterpret_cast<const float*>(pts) + 3 * i;
    x = p[0]; y = p[1]; z = p[2];
  }
}

// ---- geometry.visibility_mask (geometry.py:89-103): thread per (point, view) -----------------------
template <int PT>
__global__ void k_visibility_mask(const void* __restrict__ pts, int64_t n,
                                  const pf_view_t* __restrict__ views, int nv,
                                  const float* __restrict__ depth, double eps,
                                  uint8_t* __restrict__ mask) {
  extern __shared__ pf_view_t s_views[];
  for (int j = threadIdx.x; j < nv; j += blockDim.x) s_views[j] = views[j];
  __syncthreads();
  const int64_t total = n * nv;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nv;
    const int j = (int)(e - i * nv);
    double x, y, z;
    load_point<PT>(pts, i, x, y, z);
    const pf_view_t& vw = s_views[j];
    const Proj q = project(vw, x, y, z);
    mask[e] = depth_test(depth + vw.depth_offset, vw.H, vw.W, q.u, q.v, q.z, eps) ? 1 : 0;
  }
}

// ---- fusion.aggregate_geometric_features (fusion.py:65-93) ---------------------------------------
// warp per point; per channel the fp64 accumulation runs over views in view order starting from
// 0.0 exactly like `accum[rows] += sampled` (fusion.py:75-87), then one division (fusion.py:89-90).
template <int PT, int DT>
__global__ void k_aggregate(const void* __restrict__ pts, int64_t n,
                            const pf_view_t* __restrict__ views, int nv,
                            const void* __restrict__ fmap, int d,
                            const uint8_t* __restrict__ vis, double* __restrict__ feats,
                            int64_t* __restrict__ counts) {
  extern __shared__ pf_view_t s_views[];
  for (int j = threadIdx.x; j < nv; j += blockDim.x) s_views[j] = views[j];
  __syncthreads();
  constexpr int CH = 8;  // channels per lane per chunk
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n;
       i += warps) {
    double x, y, z;
    load_point<PT>(pts, i, x, y, z);
    int64_t cnt = 0;
    for (int j = 0; j < nv; ++j) cnt += vis[i * nv + j] ? 1 : 0;
    for (int c0 = 0; c0 < d; c0 += 32 * CH) {
      double acc[CH];
#pragma unroll
      for (int q = 0; q < CH; ++q) acc[q] = 0.0;
      for (int j = 0; j < nv; ++j) {
        if (!vis[i * nv + j]) continue;
        const pf_view_t& vw = s_views[j];
        const Proj q = project(vw, x, y, z);
        const double ratio_u = (double)vw.Wf / (double)vw.W;
        const double ratio_v = (double)vw.Hf / (double)vw.H;
        const Taps t = make_taps(feat_coord(q.u, ratio_u), feat_coord(q.v, ratio_v), vw.Hf, vw.Wf);
        const char* base = reinterpret_cast<const char*>(fmap) +
                           vw.fmap_offset * (DT == PF_F32 ? 4 : 2);
#pragma unroll
        for (int qq = 0; qq < CH; ++qq) {
          const int c = c0 + qq * 32 + lane;
          if (c < d) acc[qq] = __dadd_rn(acc[qq], bilinear_sample<DT>(base, t, vw.Wf, d, c));
        }
      }
#pragma unroll
      for (int qq = 0; qq < CH; ++qq) {
        const int c = c0 + qq * 32 + lane;
        if (c < d) feats[i * d + c] = cnt > 0 ? __ddiv_rn(acc[qq], (double)cnt) : 0.0;
      }
    }
    if (lane == 0) counts[i] = cnt;
  }
}

// ---- grounding.material_similarity (grounding.py:158-165): f64 tiled GEMM f @ text^T ----------------
constexpr int SIM_TS = 32;  // rows per block
constexpr int SIM_TK = 32;  // materials per block
constexpr int SIM_TD = 32;  // reduction chunk

__global__ void k_similarity(const double* __restrict__ f, int64_t s, int d,
                             const double* __restrict__ t, int k, double* __restrict__ out) {
  __shared__ double sf[SIM_TS][SIM_TD + 1];
  __shared__ double st[SIM_TK][SIM_TD + 1];
  const int tx = threadIdx.x & 31;  // material within tile
  const int ty = threadIdx.x >> 5;  // 8 warps, 4 rows each
  const int64_t r0 = blockIdx.x * (int64_t)SIM_TS;
  const int k0 = blockIdx.y * SIM_TK;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int d0 = 0; d0 < d; d0 += SIM_TD) {
    for (int e = threadIdx.x; e < SIM_TS * SIM_TD; e += blockDim.x) {
      const int rr = e / SIM_TD, cc = e % SIM_TD;
      const int64_t row = r0 + rr;
      sf[rr][cc] = (row < s && d0 + cc < d) ? f[row * d + d0 + cc] : 0.0;
      const int kk = k0 + rr;
      st[rr][cc] = (kk < k && d0 + cc < d) ? t[(int64_t)kk * d + d0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < SIM_TD; ++cc) {
      const double tv = st[tx][cc];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(sf[ty * 4 + q][cc], tv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t row = r0 + ty * 4 + q;
    if (row < s && k0 + tx < k) out[row * k + k0 + tx] = acc[q];
  }
}

// ---- grounding.softmax_weights (grounding.py:168-178): warp per row --------------------------------
__global__ void k_softmax(const double* __restrict__ sims, int64_t s, int k, double temp,
                          const uint8_t* __restrict__ row_valid, double* __restrict__ w,
                          int32_t* __restrict__ nan_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < s;
       i += warps) {
    const double* row = sims + i * k;
    double* wr = w + i * k;
    if (row_valid && !row_valid[i]) {
      for (int c = lane; c < k; c += 32) wr[c] = 0.0;
      continue;
    }
    double m = -INFINITY;
    bool nan = false;
    for (int c = lane; c < k; c += 32) {
      const double v = row[c];
      nan |= isnan(v);
      m = fmax(m, __ddiv_rn(v, temp));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (__any_sync(0xffffffffu, nan) && lane == 0) atomicOr(nan_flag, 1);
    double sum = 0.0;
    for (int c = lane; c < k; c += 32) {
      const double e = exp(__dsub_rn(__ddiv_rn(row[c], temp), m));
      wr[c] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    for (int c = lane; c < k; c += 32) wr[c] = __ddiv_rn(wr[c], sum);
  }
}

// ---- grounding.regress_with_weights (grounding.py:198-202) ----------------------------------------
__global__ void k_regress(const double* __restrict__ w, int64_t s, int k,
                          const double* __restrict__ y, int p, double* __restrict__ out) {
  const int64_t total = s * p;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / p;
    const int c = (int)(e - i * p);
    double acc = 0.0;
    for (int q = 0; q < k; ++q) acc = fma(w[i * k + q], y[(int64_t)q * p + c], acc);
    out[e] = acc;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int pf_visible_in_view(const double* u, const double* v, const double* z, int64_t n,
                       const float* depth, int32_t h, int32_t w, double eps, uint8_t* out,
                       void* stream) {
  if (n < 0 || h < 0 || w < 0) return set_error(PF_ERR_VALUE, "visible_in_view: negative size");
  if (n == 0) return PF_OK;
  k_visible_in_view<<<grid_for(n, 256), 256, 0, S(stream)>>>(u, v, z, n, depth, h, w, eps, out);
  return check_launch("visible_in_view");
}

static int gather_common(const void* fmap, int32_t dt, int32_t hf, int32_t wf, int32_t d,
                         const double* fu, const double* fv, const int64_t* rows, int64_t m,
                         double* out, int64_t* counts, void* stream, bool accum) {
  if (hf <= 0 || wf <= 0 || d <= 0)
    return set_error(PF_ERR_STRUCTURE, "feature map must be (Hf, Wf, D) with positive sizes");
  if (dt != PF_F32 && dt != PF_BF16) return set_error(PF_ERR_VALUE, "fmap dtype must be f32|bf16");
  if (m <= 0) return PF_OK;
  const int blocks = grid_for(m * 32, 256);
  if (dt == PF_F32) {
    if (accum)
      k_gather<PF_F32, true><<<blocks, 256, 0, S(stream)>>>(fmap, hf, wf, d, fu, fv, m, rows, out, counts);
    else
      k_gather<PF_F32, false><<<blocks, 256, 0, S(stream)>>>(fmap, hf, wf, d, fu, fv, m, rows, out, counts);
  } else {
    if (accum)
      k_gather<PF_BF16, true><<<blocks, 256, 0, S(stream)>>>(fmap, hf, wf, d, fu, fv, m, rows, out, counts);
    else
      k_gather<PF_BF16, false><<<blocks, 256, 0, S(stream)>>>(fmap, hf, wf, d, fu, fv, m, rows, out, counts);
  }
  return check_launch(accum ? "accumulate_features" : "bilinear_gather");
}

int pf_bilinear_gather(const void* fmap, int32_t dt, int32_t hf, int32_t wf, int32_t d,
                       const double* fu, const double* fv, int64_t m, double* out, void* stream) {
  return gather_common(fmap, dt, hf, wf, d, fu, fv, nullptr, m, out, nullptr, stream, false);
}

int pf_accumulate_features(const void* fmap, int32_t dt, int32_t hf, int32_t wf, int32_t d,
                           const double* fu, const double* fv, const int64_t* rows, int64_t m,
                           double* accum, int64_t* counts, void* stream) {
  return gather_common(fmap, dt, hf, wf, d, fu, fv, rows, m, accum, counts, stream, true);
}

int pf_project_points(const double* points, int64_t n, const pf_view_t* view_host, double* uv,
                      double* z, void* stream) {
  if (!view_host) return set_error(PF_ERR_VALUE, "project_points: null view");
  if (n <= 0) return PF_OK;
  k_project<<<grid_for(n, 256), 256, 0, S(stream)>>>(points, n, *view_host, uv, z);
  return check_launch("project_points");
}

int pf_visibility_mask(const void* points, int32_t pdt, int64_t n, const pf_view_t* views,
                       int32_t nv, const float* depth, double eps, uint8_t* mask, void* stream) {
  if (nv <= 0) return set_error(PF_ERR_STRUCTURE, "visibility_mask: no views");
  if (pdt != PF_F32 && pdt != PF_F64) return set_error(PF_ERR_VALUE, "points must be f32|f64");
  if (n <= 0) return PF_OK;
  const size_t smem = sizeof(pf_view_t) * (size_t)nv;
  if (smem > 200 * 1024) return set_error(PF_ERR_STRUCTURE, "too many views (%d)", nv);
  const int blocks = grid_for(n * nv, 256);
  if (pdt == PF_F64) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_visibility_mask<PF_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_visibility_mask<PF_F64><<<blocks, 256, smem, S(stream)>>>(points, n, views, nv, depth, eps, mask);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_visibility_mask<PF_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_visibility_mask<PF_F32><<<blocks, 256, smem, S(stream)>>>(points, n, views, nv, depth, eps, mask);
  }
  return check_launch("visibility_mask");
}

int pf_aggregate_features(const void* points, int32_t pdt, int64_t n, const pf_view_t* views,
                          int32_t nv, const void* fmap, int32_t dt, int32_t d,
                          const uint8_t* vis, double* feats, int64_t* counts, void* stream) {
  if (nv <= 0) return set_error(PF_ERR_STRUCTURE, "aggregate: no views");
  if (d <= 0) return set_error(PF_ERR_STRUCTURE, "aggregate: feature dim must be positive");
  if (pdt != PF_F32 && pdt != PF_F64) return set_error(PF_ERR_VALUE, "points must be f32|f64");
  if (dt != PF_F32 && dt != PF_BF16) return set_error(PF_ERR_VALUE, "fmap dtype must be f32|bf16");
  if (n <= 0) return PF_OK;
  const size_t smem = sizeof(pf_view_t) * (size_t)nv;
  if (smem > 200 * 1024) return set_error(PF_ERR_STRUCTURE, "too many views (%d)", nv);
  const int blocks = grid_for(n * 32, 256);
#define PF_AGG(PT, DT)                                                                           \
  do {                                                                                           \
    if (smem > 48 * 1024)                                                                        \
      cudaFuncSetAttribute(k_aggregate<PT, DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                           (int)smem);                                                           \
    k_aggregate<PT, DT><<<blocks, 256, smem, S(stream)>>>(points, n, views, nv, fmap, d, vis,    \
                                                          feats, counts);                        \
  } while (0)
  if (pdt == PF_F64) {
    if (dt == PF_F32) PF_AGG(PF_F64, PF_F32); else PF_AGG(PF_F64, PF_BF16);
  } else {
    if (dt == PF_F32) PF_AGG(PF_F32, PF_F32); else PF_AGG(PF_F32, PF_BF16);
  }
#undef PF_AGG
  return check_launch("aggregate_geometric_features");
}

int pf_material_similarity(const double* f, int64_t s, int32_t d, const double* t, int32_t k,
                           double* out, void* stream) {
  if (d <= 0 || k <= 0) return set_error(PF_ERR_STRUCTURE, "similarity: bad shapes d=%d k=%d", d, k);
  if (s <= 0) return PF_OK;
  dim3 grid((unsigned)((s + SIM_TS - 1) / SIM_TS), (unsigned)((k + SIM_TK - 1) / SIM_TK));
  k_similarity<<<grid, 256, 0, S(stream)>>>(f, s, d, t, k, out);
  return check_launch("material_similarity");
}

int pf_softmax_weights(const double* sims, int64_t s, int32_t k, double temperature,
                       const uint8_t* row_valid, double* w, int32_t* nan_flag, void* stream) {
  if (!(temperature > 0.0))
    return set_error(PF_ERR_VALUE, "temperature must be positive, got %g", temperature);
  if (k <= 0) return set_error(PF_ERR_STRUCTURE, "softmax: k must be positive");
  if (s <= 0) return PF_OK;
  k_softmax<<<grid_for(s * 32, 256), 256, 0, S(stream)>>>(sims, s, k, temperature, row_valid, w,
                                                          nan_flag);
  return check_launch("softmax_weights");
}

int pf_regress_with_weights(const double* w, int64_t s, int32_t k, const double* y, int32_t p,
                            double* out, void* stream) {
  if (k <= 0 || p <= 0) return set_error(PF_ERR_STRUCTURE, "regress: bad shapes k=%d p=%d", k, p);
  if (s <= 0) return PF_OK;
  k_regress<<<grid_for(s * p, 256), 256, 0, S(stream)>>>(w, s, k, y, p, out);
  return check_launch("regress_with_weights");
}

}  // extern "C"

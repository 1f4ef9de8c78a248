// The fused fusion + property-query path, SIMT version for sm_100a.
//
// One warp owns one point at a time (persistent grid, warps stride over points):
//   1. lanes over views: fp64 projection + nearest-pixel depth test (geometry.py:89-103 /
//      numpy_impl.py:14-40, bit-exact), bilinear tap geometry (fusion.py:83-86,
//      numpy_impl.py:50-57); a ballot gives the visibility bitset word, visible taps are compacted
//      into a per-warp shared-memory list;
//   2. lanes over channels: for every visible view the 4 taps are read with 16-byte coalesced
//      loads from the channel-last map and accumulated in fp32 registers (accumulate_features,
//      numba_impl.py:63-89). The 1/count of the mean (fusion.py:89-90) cancels in the
//      normalisation and is only applied when features are written for validation;
//   3. cosine similarity by associativity: s_ik = <F_i, t_k>/|F_i| with F_i = sum_taps w * f_tap,
//      so <F_i, t_k> = sum_taps w * G[tap, k] where G = fmap @ text^T is precomputed once per call
//      (k_text_proj) — each lane accumulates its materials alongside the channel gather, and |F_i|
//      comes from a warp reduction of the channel accumulators (fusion.py:210-214 normalisation
//      rule; grounding.py:158-165);
//   4. temperature softmax across lanes (grounding.py:168-178), property regression
//      (grounding.py:198-202), voxel code + dense voxel partials, and the
//      integrate_mass partial sums (integrate.py:133-155), reduced per block then atomically.
// Featureless points (count 0) get zero probability / property rows (pipeline.py:279-280).
#include <climits>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "pf_common.cuh"
#include "pf_tile.cuh"

namespace pf {
namespace {

constexpr int kFuseThreads = 256;
constexpr int kFuseWarps = kFuseThreads / 32;
constexpr int kMaxKpl = 8;  // materials per lane -> k <= 256
constexpr int kMaxP = 4;

// ---- G = fmap @ text^T over every cell of every view (fp32 SIMT tiled GEMM) ------------------------
constexpr int TP_CELLS = 64, TP_MATS = 32, TP_D = 32;

template <int DT>
__global__ void __launch_bounds__(256) k_text_proj(const void* __restrict__ fmap, int64_t cells,
                                                   int d, const float* __restrict__ text, int k,
                                                   int kpad, float* __restrict__ G) {
  __shared__ float sa[TP_CELLS][TP_D + 1];
  __shared__ float sb[TP_MATS][TP_D + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c0 = blockIdx.x * (int64_t)TP_CELLS;
  const int m0 = blockIdx.y * TP_MATS;
  float acc[TP_CELLS / 8];
#pragma unroll
  for (int q = 0; q < TP_CELLS / 8; ++q) acc[q] = 0.f;
  for (int d0 = 0; d0 < d; d0 += TP_D) {
    for (int e = threadIdx.x; e < TP_CELLS * TP_D; e += blockDim.x) {
      const int r = e / TP_D, c = e % TP_D;
      sa[r][c] = (c0 + r < cells && d0 + c < d) ? load_feat<DT>(fmap, (c0 + r) * d + d0 + c) : 0.f;
    }
    for (int e = threadIdx.x; e < TP_MATS * TP_D; e += blockDim.x) {
      const int r = e / TP_D, c = e % TP_D;
      sb[r][c] = (m0 + r < k && d0 + c < d) ? __ldg(text + (int64_t)(m0 + r) * d + d0 + c) : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int c = 0; c < TP_D; ++c) {
      const float b = sb[tx][c];
#pragma unroll
      for (int q = 0; q < TP_CELLS / 8; ++q) acc[q] = fmaf(sa[ty * (TP_CELLS / 8) + q][c], b, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < TP_CELLS / 8; ++q) {
    const int64_t cell = c0 + ty * (TP_CELLS / 8) + q;
    if (cell < cells && m0 + tx < kpad) G[cell * kpad + m0 + tx] = acc[q];
  }
}

struct FuseParams {
  const float* points;
  int64_t n;
  const pf_view_t* views;
  int nv, nwords;
  const float* depth;
  const void* fmap;
  int d;
  const float* G;
  int k, kpl, kpad;
  const float* values;
  int p, density_col;
  const float* mid_theta;
  float inv_temp;
  double eps;
  int grid;
  const double* lo_hi;
  uint32_t flags;
  int32_t* counts;
  uint32_t* mask_bits;
  float* props;
  int32_t* codes;
  float* grid_partials;
  int32_t* vox_list;   // optional touched-voxel list
  int32_t* vox_count;
  int64_t vox_base;    // first list slot of this kernel (n when the tile path owns slots 0..n-1)
  double* partials;
  int32_t* status;
  float* features;
  float* sims;
  float* weights;
  const int32_t* list;      // optional: process only these point indices (tile-path overflow)
  const int32_t* list_len;  // device count of `list`
};

struct __align__(16) TapEntry {
  int32_t c00;    // global cell index of (y0, x0)
  int32_t dyxw;   // (dyW << 1) | dx : offsets to the other three taps
  float wx, wy;
};

// load VEC consecutive channels starting at element `idx` of a map of dtype DT, as fp32
template <int DT, int VEC>
__device__ __forceinline__ void load_vec(const void* base, int64_t idx, float* out) {
  if constexpr (VEC == 1) {
    out[0] = load_feat<DT>(base, idx);
  } else if constexpr (DT == PF_F32) {
    static_assert(VEC == 4, "f32 vector loads are float4");
    const float4 v = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + idx));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else {
    static_assert(VEC == 8, "bf16 vector loads are 8 x bf16");
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(base) + idx));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      out[2 * q] = __uint_as_float(w[q] << 16);
      out[2 * q + 1] = __uint_as_float(w[q] & 0xffff0000u);
    }
  }
}

// channel index of element (chunk j, element e) owned by `lane`
template <int VEC>
__device__ __forceinline__ int chan(int j, int e, int lane) {
  return j * 32 * VEC + lane * VEC + e;
}

template <int DT, int VEC, int NCHUNK>
__global__ void __launch_bounds__(kFuseThreads, 3) k_fuse_simt(FuseParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  pf_view_t* s_views = reinterpret_cast<pf_view_t*>(smem);
  float* s_vals = reinterpret_cast<float*>(s_views + P.nv);       // [kpad][kMaxP]
  float* s_mt = s_vals + P.kpad * kMaxP;                            // [kpad]
  double* s_red = reinterpret_cast<double*>(s_mt + P.kpad);         // [kpad + 6]
  TapEntry* s_taps = reinterpret_cast<TapEntry*>(s_red + P.kpad + 8);  // [warps][nv]

  for (int j = threadIdx.x; j < P.nv; j += blockDim.x) s_views[j] = P.views[j];
  for (int j = threadIdx.x; j < P.kpad * kMaxP; j += blockDim.x) {
    const int kk = j / kMaxP, pp = j % kMaxP;
    s_vals[j] = (kk < P.k && pp < P.p) ? P.values[kk * P.p + pp] : 0.f;
  }
  for (int j = threadIdx.x; j < P.kpad; j += blockDim.x) s_mt[j] = j < P.k ? P.mid_theta[j] : 0.f;
  for (int j = threadIdx.x; j < P.kpad + 8; j += blockDim.x) s_red[j] = 0.0;
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TapEntry* my_taps = s_taps + warp * P.nv;
  double lo[3];
  const double edge = voxel_edge(P.lo_hi, P.grid, lo);
  const bool do_vox = !(P.flags & PF_FUSE_SKIP_VOXELS);
  const int64_t cells3 = (int64_t)P.grid * P.grid * P.grid;

  double wt[kMaxKpl];
#pragma unroll
  for (int q = 0; q < kMaxKpl; ++q) wt[q] = 0.0;
  double pm_sum = 0.0, pmx = 0.0, pmy = 0.0, pmz = 0.0, featured = 0.0, pairs = 0.0;

  constexpr int CPL = VEC * NCHUNK;
  const int64_t nwarps = (int64_t)gridDim.x * kFuseWarps;
  const int64_t total = P.list ? (int64_t)*P.list_len : P.n;
  for (int64_t t = blockIdx.x * (int64_t)kFuseWarps + warp; t < total; t += nwarps) {
    const int64_t i = P.list ? (int64_t)P.list[t] : t;
    const float px = __ldg(P.points + 3 * i), py = __ldg(P.points + 3 * i + 1),
                pz = __ldg(P.points + 3 * i + 2);
    // ---- phase 1: lanes over views -----------------------------------------------------------
    int count = 0;
    for (int vb = 0; vb < P.nwords; ++vb) {
      const int v = vb * 32 + lane;
      bool vis = false;
      TapEntry te;
      if (v < P.nv) {
        const pf_view_t& vw = s_views[v];
        const Proj q = project(vw, (double)px, (double)py, (double)pz);
        vis = depth_test(P.depth + vw.depth_offset, vw.H, vw.W, q.u, q.v, q.z, P.eps);
        if (vis) {
          const Taps t = make_taps(feat_coord(q.u, (double)vw.Wf / (double)vw.W),
                                   feat_coord(q.v, (double)vw.Hf / (double)vw.H), vw.Hf, vw.Wf);
          te.c00 = (int32_t)(vw.fmap_offset / P.d) + t.y0 * vw.Wf + t.x0;
          te.dyxw = (((t.y1 - t.y0) * vw.Wf) << 1) | (t.x1 - t.x0);
          te.wx = (float)t.wx;
          te.wy = (float)t.wy;
        }
      }
      const uint32_t bits = __ballot_sync(0xffffffffu, vis);
      if (vis) my_taps[count + __popc(bits & ((1u << lane) - 1u))] = te;
      if (lane == 0) P.mask_bits[i * P.nwords + vb] = bits;
      count += __popc(bits);
    }
    __syncwarp();
    // ---- phase 2: lanes over channels (+ materials) -----------------------------------------------
    float acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.f;
    float gacc[kMaxKpl];
#pragma unroll
    for (int q = 0; q < kMaxKpl; ++q) gacc[q] = 0.f;
    for (int e = 0; e < count; ++e) {
      const TapEntry te = my_taps[e];
      const int dx = te.dyxw & 1, dyw = te.dyxw >> 1;
      const float w00 = (1.f - te.wy) * (1.f - te.wx), w01 = (1.f - te.wy) * te.wx;
      const float w10 = te.wy * (1.f - te.wx), w11 = te.wy * te.wx;
      const int64_t c00 = te.c00, c01 = c00 + dx, c10 = c00 + dyw, c11 = c10 + dx;
#pragma unroll
      for (int j = 0; j < NCHUNK; ++j) {
        const int ch = chan<VEC>(j, 0, lane);
        if (VEC > 1 || ch < P.d) {
          float f00[VEC], f01[VEC], f10[VEC], f11[VEC];
          load_vec<DT, VEC>(P.fmap, c00 * P.d + ch, f00);
          load_vec<DT, VEC>(P.fmap, c01 * P.d + ch, f01);
          load_vec<DT, VEC>(P.fmap, c10 * P.d + ch, f10);
          load_vec<DT, VEC>(P.fmap, c11 * P.d + ch, f11);
#pragma unroll
          for (int q = 0; q < VEC; ++q) {
            float a = acc[j * VEC + q];
            a = fmaf(w00, f00[q], a);
            a = fmaf(w01, f01[q], a);
            a = fmaf(w10, f10[q], a);
            a = fmaf(w11, f11[q], a);
            acc[j * VEC + q] = a;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) {
        if (q < P.kpl) {
          const int kk = lane + 32 * q;
          float g = gacc[q];
          g = fmaf(w00, __ldg(P.G + c00 * P.kpad + kk), g);
          g = fmaf(w01, __ldg(P.G + c01 * P.kpad + kk), g);
          g = fmaf(w10, __ldg(P.G + c10 * P.kpad + kk), g);
          g = fmaf(w11, __ldg(P.G + c11 * P.kpad + kk), g);
          gacc[q] = g;
        }
      }
    }
    __syncwarp();
    // ---- phase 3: normalise, similarity, softmax, regression --------------------------------------
    float ss = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c) ss = fmaf(acc[c], acc[c], ss);
    const float norm2 = warp_sum(ss);
    if ((P.flags & PF_FUSE_WRITE_FEATURES) && P.features) {
      const float invc = count > 0 ? 1.f / (float)count : 0.f;
#pragma unroll
      for (int j = 0; j < NCHUNK; ++j) {
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
          const int ch = chan<VEC>(j, q, lane);
          if (ch < P.d) P.features[i * P.d + ch] = acc[j * VEC + q] * invc;
        }
      }
    }
    float w[kMaxKpl];
    float prop[kMaxP] = {0.f, 0.f, 0.f, 0.f};
    float pm = 0.f;
    if (count > 0) {
      // fusion.py:210-214: normalise only when |f| > 0 (a zero vector stays zero)
      const float inv = norm2 > 0.f ? 1.f / sqrtf(norm2) : 0.f;
      float m = -INFINITY;
      bool nan = false;
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) {
        const int kk = lane + 32 * q;
        const bool valid = q < P.kpl && kk < P.k;
        const float s = gacc[q] * inv;
        w[q] = valid ? s : 0.f;  // holds the similarity until the softmax below
        if (valid) {
          nan |= isnan(s);
          m = fmaxf(m, s * P.inv_temp);
        }
      }
      if (__any_sync(0xffffffffu, nan) && lane == 0) atomicOr(P.status, 1);
      m = warp_max(m);
      if ((P.flags & PF_FUSE_WRITE_SIMS) && P.sims) {
#pragma unroll
        for (int q = 0; q < kMaxKpl; ++q) {
          const int kk = lane + 32 * q;
          if (q < P.kpl && kk < P.k) P.sims[i * P.k + kk] = w[q];
        }
      }
      float se = 0.f;
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) {
        const int kk = lane + 32 * q;
        const bool valid = q < P.kpl && kk < P.k;
        const float e = valid ? expf(w[q] * P.inv_temp - m) : 0.f;
        w[q] = e;
        se += e;
      }
      const float se_t = warp_sum(se);
      // a non-finite sum without a NaN similarity means infinite inputs: flag it (bit 1) rather than
      // return NaN properties silently
      if (lane == 0 && !(se_t <= 3.4e38f)) atomicOr(P.status, 2);
      const float rs = 1.f / se_t;
      float pl[kMaxP] = {0.f, 0.f, 0.f, 0.f};
      float pml = 0.f;
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) {
        const int kk = lane + 32 * q;
        if (q < P.kpl) {
          w[q] *= rs;
#pragma unroll
          for (int pp = 0; pp < kMaxP; ++pp) pl[pp] = fmaf(w[q], s_vals[kk * kMaxP + pp], pl[pp]);
          pml = fmaf(w[q], s_mt[kk], pml);
          wt[q] += (double)w[q];
        }
      }
#pragma unroll
      for (int pp = 0; pp < kMaxP; ++pp) prop[pp] = pp < P.p ? warp_sum(pl[pp]) : 0.f;
      pm = warp_sum(pml);
    } else {
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) w[q] = 0.f;
      if ((P.flags & PF_FUSE_WRITE_SIMS) && P.sims) {
#pragma unroll
        for (int q = 0; q < kMaxKpl; ++q) {
          const int kk = lane + 32 * q;
          if (q < P.kpl && kk < P.k) P.sims[i * P.k + kk] = 0.f;
        }
      }
    }
    if ((P.flags & PF_FUSE_WRITE_WEIGHTS) && P.weights) {
#pragma unroll
      for (int q = 0; q < kMaxKpl; ++q) {
        const int kk = lane + 32 * q;
        if (q < P.kpl && kk < P.k) P.weights[i * P.k + kk] = w[q];
      }
    }
    if (lane < P.p) {
      float pv = prop[0];
#pragma unroll
      for (int pp = 1; pp < kMaxP; ++pp) pv = lane == pp ? prop[pp] : pv;
      P.props[i * P.p + lane] = pv;
    }
    if (lane == 0) {
      P.counts[i] = count;
      // a NaN point is a padding slot of the fixed-capacity sharded exchange (pf_shard_pack_padded):
      // it projects nowhere (count 0, zero outputs), has voxel code -1 and no voxel contribution
      const int32_t code = isnan(px) ? -1 : voxel_code(px, py, pz, lo, edge, P.grid);
      P.codes[i] = code;
      if (do_vox && code >= 0) {
        float rho = prop[0];
#pragma unroll
        for (int pp = 1; pp < kMaxP; ++pp) rho = P.density_col == pp ? prop[pp] : rho;
        atomicAdd(P.grid_partials + code, rho);
        // touched-voxel list: the SIMT points append after the tile path's n slots
        if (atomicAdd(P.grid_partials + cells3 + code, 1.0f) == 0.0f && P.vox_list)
          P.vox_list[P.vox_base + atomicAdd(P.vox_count, 1)] = code;
      }
      if (code >= 0) {  // padding slots (NaN coordinates) stay out of the integrate partials
        pm_sum += pm;
        pmx += (double)pm * px;
        pmy += (double)pm * py;
        pmz += (double)pm * pz;
        featured += count > 0 ? 1.0 : 0.0;
        pairs += count;
      }
    }
  }
  // ---- block + grid reduction of the integrate_mass partials ---------------------------------------
#pragma unroll
  for (int q = 0; q < kMaxKpl; ++q) {
    const int kk = lane + 32 * q;
    if (q < P.kpl && kk < P.k && wt[q] != 0.0) atomicAdd(s_red + kk, wt[q]);
  }
  if (lane == 0) {
    atomicAdd(s_red + P.k + 0, pm_sum);
    atomicAdd(s_red + P.k + 1, pmx);
    atomicAdd(s_red + P.k + 2, pmy);
    atomicAdd(s_red + P.k + 3, pmz);
    atomicAdd(s_red + P.k + 4, featured);
    atomicAdd(s_red + P.k + 5, pairs);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < P.k + 6; j += blockDim.x)
    if (s_red[j] != 0.0) atomicAdd(P.partials + j, s_red[j]);
}

struct Occ {
  std::once_flag once;
  int blocks_per_sm = 1;
  int sms = 148;
};

template <int DT, int VEC, int NCHUNK>
int launch_fuse(const FuseParams& prm, size_t smem, cudaStream_t st) {
  static Occ occ;
  auto kern = k_fuse_simt<DT, VEC, NCHUNK>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::call_once(occ.once, [&] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&occ.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ.blocks_per_sm, kern, kFuseThreads, smem);
    if (occ.blocks_per_sm < 1) occ.blocks_per_sm = 1;
  });
  int64_t want = prm.list ? INT64_MAX : (prm.n + kFuseWarps - 1) / kFuseWarps;
  int64_t cap = (int64_t)occ.sms * occ.blocks_per_sm;
  int blocks = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  kern<<<blocks, kFuseThreads, smem, st>>>(prm);
  return check_launch("fuse_query_simt");
}

}  // namespace
}  // namespace pf

using namespace pf;

namespace {
// one forked stream (+ fork / join events) per host thread and device: a stream shared between
// threads could start one caller's prepare at another caller's fork point
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
constexpr int kMaxDevices = 64;

SideStream* side_stream() {
  static thread_local SideStream per_dev[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  SideStream& x = per_dev[dev];
  if (!x.s) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (getenv("PF_SIDE_LOWPRI")) hi = lo;  // A/B knob: the forked stream at the default priority
    if (cudaStreamCreateWithPriority(&x.s, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x = SideStream{};
      return nullptr;  // run the prepare inline on the caller's stream
    }
  }
  return &x;
}
}  // namespace

extern "C" int pf_fuse_prepare(const pf_fuse_args_t* a, void* stream);

namespace {
// ForkHook of pf_fuse_query: the per-object tables on the forked stream, after the point sort
cudaEvent_t fork_prepare(void* ctx, cudaStream_t st, int* rc) {
  SideStream* side = side_stream();
  const pf_fuse_args_t* a = static_cast<const pf_fuse_args_t*>(ctx);
  if (!side) {
    if (a->fmap_ready) cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(a->fmap_ready), 0);
    *rc = pf_fuse_prepare(a, st);
    return nullptr;
  }
  cudaEventRecord(side->fork, st);
  cudaStreamWaitEvent(side->s, side->fork, 0);
  if (a->fmap_ready) cudaStreamWaitEvent(side->s, static_cast<cudaEvent_t>(a->fmap_ready), 0);
  *rc = pf_fuse_prepare(a, side->s);
  cudaEventRecord(side->join, side->s);
  return side->join;
}
}  // namespace

extern "C" {

static int64_t total_cells(const pf_fuse_args_t* a) {
  int64_t cells = 0;
  for (int j = 0; j < a->nviews; ++j) {
    const pf_view_t& v = a->views_host[j];
    const int64_t end = v.fmap_offset / a->d + (int64_t)v.Hf * v.Wf;
    if (end > cells) cells = end;
  }
  return cells;
}

static int kpl_of(int k) { return (k + 31) / 32; }

// The tensor-core tile path (pf_tile.cu) applies to bf16 maps with D a multiple of 128, <= 64
// views, feature grids <= 255 per side and <= 128 padded materials.
// f32 maps take the tile path in x3 mode (bf16 hi/lo split operands, three MMAs per k-step)
static bool tile_x3(const pf_fuse_args_t* a) { return a->fmap_dtype == PF_F32; }

// below this many points the x3 path's fixed costs (sort, prep, operand splits) exceed the SIMT pass
constexpr int64_t kX3MinPoints = 65536;

static bool tile_path_ok(const pf_fuse_args_t* a) {
  if ((a->fmap_dtype != PF_BF16 && a->fmap_dtype != PF_F32) || a->d % 128 != 0 || a->nviews > tile::kMaxViewsTC)
    return false;
  if (a->fmap_dtype == PF_F32 && a->n < kX3MinPoints) return false;
  if (((a->k + 63) / 64) * 64 > tile::kMaxKpadTC || (a->flags & PF_FUSE_FORCE_SIMT)) return false;
  // uniform, contiguously packed views (the TMA tensor maps address them as one [V*Hf][Wf][D] block)
  const pf_view_t& v0 = a->views_host[0];
  if (v0.Hf > 255 || v0.Wf > 255) return false;
  for (int j = 0; j < a->nviews; ++j) {
    const pf_view_t& v = a->views_host[j];
    if (v.Hf != v0.Hf || v.Wf != v0.Wf || v.fmap_offset != (int64_t)j * v0.Hf * v0.Wf * a->d) return false;
  }
  return true;
}

// bf16 maps take the Gram-formulation kernel (pf_gram.cu, 512-point tiles) unless mean features are
// requested (validation output only the feature-product kernel k_tile_ws produces); PF_GRAM=0 forces
// k_tile_ws (A/B measurements)
static bool tile_gram(const pf_fuse_args_t* a) {
  static const bool off = [] {
    const char* e = getenv("PF_GRAM");
    return e && e[0] == '0';
  }();
  return !off && a->fmap_dtype == PF_BF16 && !(a->flags & (PF_FUSE_WRITE_FEATURES | PF_FUSE_FEATURE_KERNEL));
}
static int tile_rows(const pf_fuse_args_t* a) { return tile_gram(a) ? tile::kGramTile : tile::kTile; }
// Gram path: split items (128 / 32 rows) to the feature-product kernel (PF_GRAM_SPLIT=0: all items in
// the Gram kernel)
static bool gram_split() {
  static const bool split = [] {
    const char* e = getenv("PF_GRAM_SPLIT");
    return !(e && e[0] == '0');
  }();
  return split;
}

static uint64_t g_bytes(const pf_fuse_args_t* a) {
  const uint64_t g = (uint64_t)total_cells(a) * (uint64_t)(32 * kpl_of(a->k)) * sizeof(float);
  return (g + 255) & ~uint64_t(255);
}

// SIMT path over >= this many points: points are visited in Hilbert order (neighbouring warps of a
// block gather mostly the same taps, so the tap rows are served from L1 instead of L2)
constexpr int64_t kSimtOrderMin = 65536;

static uint64_t simt_order_bytes(int64_t n) {
  return ((sizeof(int32_t) * (uint64_t)n + 255) & ~uint64_t(255)) + 256 + tile::point_order_bytes(n);
}

uint64_t pf_fuse_workspace_bytes(const pf_fuse_args_t* a) {
  if (!a || !a->views_host || a->d <= 0 || a->k <= 0) return 0;
  uint64_t bytes = g_bytes(a);
  if (tile_path_ok(a)) {
    // sized for either tile kernel: a buffer set may be reused with and without feature outputs
    const uint64_t b128 = tile::tile_layout(a->n, a->nviews, total_cells(a), tile::kMaxKpadTC, a->d, tile_x3(a)).bytes;
    const uint64_t b512 = tile_x3(a) ? 0 : tile::tile_layout(a->n, a->nviews, total_cells(a), tile::kMaxKpadTC, a->d,
                                                             false, tile::kGramTile).bytes;
    bytes += b128 > b512 ? b128 : b512;
  }
  else if (a->n >= kSimtOrderMin)
    bytes += simt_order_bytes(a->n);
  return bytes;
}

static int validate(const pf_fuse_args_t* a) {
  if (!a) return set_error(PF_ERR_VALUE, "fuse_query: null args");
  if (a->n < 0) return set_error(PF_ERR_VALUE, "fuse_query: negative point count");
  if (a->nviews < 1 || a->nviews > 256)
    return set_error(PF_ERR_STRUCTURE, "fuse_query: need 1..256 views, got %d", a->nviews);
  if (!a->views_host || !a->views) return set_error(PF_ERR_VALUE, "fuse_query: views missing");
  if (a->d < 1 || a->d > 1024)
    return set_error(PF_ERR_STRUCTURE, "fuse_query: feature dim must be in [1, 1024], got %d", a->d);
  if (a->k < 1 || a->k > 32 * kMaxKpl)
    return set_error(PF_ERR_STRUCTURE, "fuse_query: need 1..256 materials, got %d", a->k);
  if (a->p < 1 || a->p > kMaxP)
    return set_error(PF_ERR_STRUCTURE, "fuse_query: need 1..4 properties, got %d", a->p);
  if (a->density_col < 0 || a->density_col >= a->p)
    return set_error(PF_ERR_VALUE, "fuse_query: density column %d out of range", a->density_col);
  if (!(a->temperature > 0.0))
    return set_error(PF_ERR_VALUE, "temperature must be positive, got %g", a->temperature);
  if (a->grid < 1 || a->grid > 1290)
    return set_error(PF_ERR_VALUE, "voxel grid side must be in [1, 1290], got %d", a->grid);
  if (a->fmap_dtype != PF_F32 && a->fmap_dtype != PF_BF16)
    return set_error(PF_ERR_VALUE, "feature maps must be f32 or bf16");
  for (int j = 0; j < a->nviews; ++j) {
    const pf_view_t& v = a->views_host[j];
    if (v.fmap_offset % a->d != 0)
      return set_error(PF_ERR_STRUCTURE, "view %d: feature offset not a multiple of D", j);
    if (v.H < 1 || v.W < 1 || v.Hf < 1 || v.Wf < 1)
      return set_error(PF_ERR_STRUCTURE, "view %d: empty depth or feature map", j);
  }
  return PF_OK;
}

int pf_fuse_prepare(const pf_fuse_args_t* a, void* stream) {
  if (int rc = validate(a)) return rc;
  if (!a->workspace) return set_error(PF_ERR_VALUE, "fuse_prepare: workspace missing");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int kpad = 32 * kpl_of(a->k);
  const int64_t cells = total_cells(a);
  float* G = reinterpret_cast<float*>(a->workspace);
  uint16_t* Gbf = nullptr;
  int kpadg = 0;
  if (tile_path_ok(a) && tile_x3(a)) {
    // f32 maps: fp32 G (SIMT), then the hi / lo bf16 splits of G and of the maps
    kpadg = tile::kMaxKpadTC;
    unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace) + g_bytes(a);
    const tile::TileLayout L = tile::tile_layout(a->n, a->nviews, cells, kpadg, a->d, true);
    uint16_t* fhi = reinterpret_cast<uint16_t*>(ws + L.fhi);
    uint16_t* flo = reinterpret_cast<uint16_t*>(ws + L.flo);
    if (int rc = tile::run_split_f32(reinterpret_cast<const float*>(a->fmap), cells, a->d, a->d, a->d, fhi, flo, st))
      return rc;
    // G on the tensor cores from the same splits (hi.hi + hi.lo + lo.hi), fp32 copy for the SIMT
    // overflow points
    if (int rc = tile::run_text_bound(a->text, a->k, a->d, reinterpret_cast<float*>(ws + L.tbound), st)) return rc;
    return tile::run_gproj_tc_x3(fhi, flo, cells, a->d, a->text, a->k, kpadg, kpad,
                                 reinterpret_cast<uint16_t*>(ws + L.gbf), reinterpret_cast<uint16_t*>(ws + L.glo), G,
                                 reinterpret_cast<uint16_t*>(ws + L.textbf), reinterpret_cast<uint16_t*>(ws + L.textlo),
                                 st);
  }
  if (tile_path_ok(a)) {
    kpadg = tile::kMaxKpadTC;  // S operand is always one 128-column chunk pair
    unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace) + g_bytes(a);
    const tile::TileLayout L = tile::tile_layout(a->n, a->nviews, cells, kpadg);
    Gbf = reinterpret_cast<uint16_t*>(ws + L.gbf);
    if (int rc = tile::run_text_bound(a->text, a->k, a->d, reinterpret_cast<float*>(ws + L.tbound), st)) return rc;
    // bf16 maps: G on the tensor cores (bf16 text), fp32 copy for the SIMT overflow tiles
    const int rc = tile::run_gproj_tc(a->fmap, cells, a->d, a->text, a->k, kpadg, kpad, Gbf, G,
                                      reinterpret_cast<uint16_t*>(ws + L.textbf), st);
    if (rc >= 0) return rc;
  }
  dim3 grid((unsigned)((cells + TP_CELLS - 1) / TP_CELLS), (unsigned)(kpad / TP_MATS));
  if (a->fmap_dtype == PF_F32)
    k_text_proj<PF_F32><<<grid, 256, 0, st>>>(a->fmap, cells, a->d, a->text, a->k, kpad, G);
  else
    k_text_proj<PF_BF16><<<grid, 256, 0, st>>>(a->fmap, cells, a->d, a->text, a->k, kpad, G);
  if (int rc = check_launch("text_proj")) return rc;
  if (Gbf) return tile::run_g_bf16(G, cells, kpad, kpadg, Gbf, st);
  return PF_OK;
}

int pf_fuse_query(const pf_fuse_args_t* a, void* stream) {
  if (int rc = validate(a)) return rc;
  if (a->n == 0) return PF_OK;
  if (!a->workspace) return set_error(PF_ERR_VALUE, "fuse_query: workspace missing");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // tile path: the per-object tables (G = fmap . text^T on the tensor cores) are built on a forked
  // high-priority stream while the point sort and the tile prep run on `st` (neither reads them);
  // the tensor-core kernel joins it. Fork / join by events, so a captured `st` captures both.
  tile::ForkHook fork;
  const bool tile = tile_path_ok(a);
  cudaEvent_t depth_ready = static_cast<cudaEvent_t>(a->depth_ready);
  cudaEvent_t fmap_ready = static_cast<cudaEvent_t>(a->fmap_ready);
  if (tile) {  // staged inputs: waited on where they are first read (run_tile_path / fork_prepare)
    fork.depth_ready = depth_ready;
    fork.fmap_ready = fmap_ready;
  } else {     // SIMT path: every input is read from the first kernel on
    if (depth_ready) cudaStreamWaitEvent(st, depth_ready, 0);
    if (fmap_ready) cudaStreamWaitEvent(st, fmap_ready, 0);
  }
  if (!(a->flags & PF_FUSE_PREPARED)) {
    if (tile && side_stream()) {
      fork.fn = fork_prepare;
      fork.ctx = const_cast<pf_fuse_args_t*>(a);
    } else {
      if (tile && fmap_ready) cudaStreamWaitEvent(st, fmap_ready, 0);
      if (int rc = pf_fuse_prepare(a, stream)) return rc;
    }
  }
  const int kpl = kpl_of(a->k), kpad = 32 * kpl;
  float* G = reinterpret_cast<float*>(a->workspace);

  FuseParams prm{};
  prm.points = a->points; prm.n = a->n; prm.views = a->views; prm.nv = a->nviews;
  prm.nwords = (a->nviews + 31) / 32; prm.depth = a->depth; prm.fmap = a->fmap; prm.d = a->d;
  prm.G = G; prm.k = a->k; prm.kpl = kpl; prm.kpad = kpad; prm.values = a->values; prm.p = a->p;
  prm.density_col = a->density_col; prm.mid_theta = a->mid_theta;
  prm.inv_temp = (float)(1.0 / a->temperature); prm.eps = a->eps; prm.grid = a->grid;
  prm.lo_hi = a->lo_hi; prm.flags = a->flags; prm.counts = a->counts; prm.mask_bits = a->mask_bits;
  prm.props = a->props; prm.codes = a->codes; prm.grid_partials = a->grid_partials;
  prm.vox_list = a->vox_list; prm.vox_count = a->vox_count; prm.vox_base = 0;
  prm.partials = a->partials; prm.status = a->status; prm.features = a->features;
  prm.sims = a->sims; prm.weights = a->weights;

  const size_t smem = sizeof(pf_view_t) * a->nviews + sizeof(float) * kpad * (kMaxP + 1) +
                      sizeof(double) * (kpad + 8) + sizeof(TapEntry) * kFuseWarps * a->nviews + 16;
  const int d = a->d;
  if (tile_path_ok(a)) {
    const int64_t cells = total_cells(a);
    const int kpadg = tile::kMaxKpadTC;  // S operand is always one 128-column chunk pair
    unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace) + g_bytes(a);
    const bool x3 = tile_x3(a);
    const int tr = tile_rows(a);
    const tile::TileLayout L = tile::tile_layout(a->n, a->nviews, cells, kpadg, a->d, x3, tr);
    tile::TileParams T{};
    T.tr = tr;
    T.deterministic = (a->flags & PF_FUSE_DETERMINISTIC) ? 1 : 0;
    T.sub1_rows = tr == tile::kGramTile ? 128 : tile::kSubRows;
    T.spts = reinterpret_cast<const float4*>(ws + L.spts);
    T.inv = reinterpret_cast<const int32_t*>(ws + L.inv);
    T.srec = reinterpret_cast<tile::SRec*>(ws + L.srec);
    T.n = a->n; T.views = a->views; T.nv = a->nviews; T.nwords = (a->nviews + 31) / 32; T.d = d;
    T.depth = a->depth; T.fmap = x3 ? (const void*)(ws + L.fhi) : a->fmap;
    T.Gbf = reinterpret_cast<const uint16_t*>(ws + L.gbf);
    T.x3 = x3 ? 1 : 0;
    T.kt_max = tr == tile::kGramTile ? tile::kGramKt : tile::ws_kt_max(x3);
    T.fmap_lo = x3 ? reinterpret_cast<const uint16_t*>(ws + L.flo) : nullptr;
    T.Gbf_lo = x3 ? reinterpret_cast<const uint16_t*>(ws + L.glo) : nullptr;
    T.kpadg = kpadg; T.k = a->k; T.p = a->p; T.density_col = a->density_col;
    T.values = a->values; T.mid_theta = a->mid_theta; T.inv_temp = prm.inv_temp; T.eps = a->eps;
    T.grid = a->grid; T.cells3 = (int64_t)a->grid * a->grid * a->grid; T.lo_hi = a->lo_hi;
    T.mask_bits = a->mask_bits; T.counts = a->counts; T.codes = a->codes; T.props = a->props;
    T.grid_partials = (a->flags & PF_FUSE_SKIP_VOXELS) ? nullptr : a->grid_partials;
    T.vox_list = a->vox_list;
    T.vox_count = a->vox_count;
    T.features = (a->flags & PF_FUSE_WRITE_FEATURES) ? a->features : nullptr;
    T.sims = (a->flags & PF_FUSE_WRITE_SIMS) ? a->sims : nullptr;
    T.weights = (a->flags & PF_FUSE_WRITE_WEIGHTS) ? a->weights : nullptr;
    T.status = a->status;
    T.tile_desc = reinterpret_cast<uint2*>(ws + L.desc);
    T.tile_kt = reinterpret_cast<int32_t*>(ws + L.kt);
    T.viewf = reinterpret_cast<tile::ViewF*>(ws + L.viewf);
    T.vbound = reinterpret_cast<float4*>(ws + L.vbound);
    T.vox = reinterpret_cast<double*>(ws + L.vox);
    T.ovf_list = reinterpret_cast<int32_t*>(ws + L.ovf) + 1;
    T.ovf_count = reinterpret_cast<int32_t*>(ws + L.ovf);
    T.sub_count = reinterpret_cast<int32_t*>(ws + L.sub);
    T.sub_tiles = T.sub_count + 1;
    T.max_sub_tiles = L.max_sub_tiles;
    T.sub2_count = reinterpret_cast<int32_t*>(ws + L.sub2);
    T.sub2_items = T.sub2_count + 1;
    T.max_sub2 = L.max_sub2;
    T.work_count = tr == tile::kGramTile ? reinterpret_cast<int32_t*>(ws + L.work) : nullptr;
    T.work = tr == tile::kGramTile ? reinterpret_cast<int4*>(ws + L.work) + 1 : nullptr;
    T.work_raw = tr == tile::kGramTile ? reinterpret_cast<int4*>(ws + L.work_raw) : nullptr;
    const bool split = gram_split();
    T.wcount = tr == tile::kGramTile && split ? reinterpret_cast<int32_t*>(ws + L.wlist) : nullptr;
    T.wlist = tr == tile::kGramTile && split ? reinterpret_cast<int4*>(ws + L.wlist) + 1 : nullptr;
    T.partials = a->partials;
    T.tbound = reinterpret_cast<const float*>(ws + L.tbound);
    T.tbox = tr == tile::kGramTile ? reinterpret_cast<float4*>(ws + L.tbox) : nullptr;
    cudaEvent_t joined = nullptr;
    if (int rc = tile::run_tile_path(T, L, ws, a->points, a->n, st, fork, &joined)) {
      if (joined) cudaStreamWaitEvent(st, joined, 0);  // rejoin the fork (keeps a capture well formed)
      return rc;
    }
    // sorted records -> caller's order; then the overflow points (tiles with more taps than fit in
    // shared memory) run through the SIMT kernel, which writes their outputs directly
    if (int rc = tile::run_unsort(T, st)) return rc;
    // overflow tiles (more taps than fit in shared memory) run through the SIMT kernel
    prm.list = T.ovf_list;
    prm.list_len = T.ovf_count;
    prm.vox_base = a->n;
  } else if (a->n >= kSimtOrderMin) {
    unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace) + g_bytes(a);
    int32_t* order = reinterpret_cast<int32_t*>(ws);
    ws += (sizeof(int32_t) * (uint64_t)a->n + 255) & ~uint64_t(255);
    int32_t* len = reinterpret_cast<int32_t*>(ws);
    ws += 256;
    if (int rc = tile::run_point_order(a->points, a->n, a->lo_hi, ws, order, len, st)) return rc;
    prm.list = order;
    prm.list_len = len;
  }
  int rc;
  if (a->fmap_dtype == PF_F32) {
    if (d == 128) rc = launch_fuse<PF_F32, 4, 1>(prm, smem, st);
    else if (d == 256) rc = launch_fuse<PF_F32, 4, 2>(prm, smem, st);
    else if (d == 512) rc = launch_fuse<PF_F32, 4, 4>(prm, smem, st);
    else if (d == 768) rc = launch_fuse<PF_F32, 4, 6>(prm, smem, st);
    else if (d == 1024) rc = launch_fuse<PF_F32, 4, 8>(prm, smem, st);
    else rc = launch_fuse<PF_F32, 1, 32>(prm, smem, st);
  } else {
    if (d == 256) rc = launch_fuse<PF_BF16, 8, 1>(prm, smem, st);
    else if (d == 512) rc = launch_fuse<PF_BF16, 8, 2>(prm, smem, st);
    else if (d == 768) rc = launch_fuse<PF_BF16, 8, 3>(prm, smem, st);
    else if (d == 1024) rc = launch_fuse<PF_BF16, 8, 4>(prm, smem, st);
    else rc = launch_fuse<PF_BF16, 1, 32>(prm, smem, st);
  }
  if (prm.list && prm.vox_base > 0) stage_mark(5, st);  // tile path: the overflow stage
  return rc;
}

/* Diagnostic: tcgen05 FLOPs the last pf_fuse_query on this workspace issued in the tile kernel, read
 * back from the workspace (synchronises the stream); 0 when the SIMT path ran. Per work item with
 * ktp = taps padded to 16: k_tile_ws 2 * 128 * ktp * (D + 128) (x3: three products); the Gram
 * kernel 2 * 128 * ktp * D (block 0) [+ 2 * 128 * (ktp - 128) * D (block 1)] + per 128-row block
 * 2 * 128 * ktp * (128 + ktp). */
int pf_tile_executed_flops(const pf_fuse_args_t* a, double* flops, void* stream) {
  *flops = 0.0;
  if (!a || !a->workspace || !tile_path_ok(a) || a->n == 0) return PF_OK;
  const int64_t cells = total_cells(a);
  const bool x3 = tile_x3(a);
  const int tr = tile_rows(a);
  const tile::TileLayout L = tile::tile_layout(a->n, a->nviews, cells, tile::kMaxKpadTC, a->d, x3, tr);
  const unsigned char* ws = reinterpret_cast<const unsigned char*>(a->workspace) + g_bytes(a);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double f = 0.0;
  if (tr == tile::kGramTile) {  // the work list the Gram kernel walked
    int32_t nw = 0;
    cudaMemcpyAsync(&nw, ws + L.work, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("tile_executed_flops");
    std::vector<int4> w((size_t)std::max(nw, 1));
    if (nw) cudaMemcpy(w.data(), ws + L.work + sizeof(int4), sizeof(int4) * nw, cudaMemcpyDeviceToHost);
    for (int i = 0; i < nw; ++i) {
      const int rows = w[i].z & 0xffff, kt = w[i].z >> 16, ktp = (kt + 15) & ~15, nb = (rows + 127) / 128;
      f += 2.0 * 128.0 * ktp * a->d + (ktp > 128 ? 2.0 * 128.0 * (ktp - 128) * a->d : 0.0);
      f += (double)nb * 2.0 * 128.0 * ktp * (double)(tile::kMaxKpadTC + ktp);
    }
    // the split items the feature-product kernel ran from its list (M = 128 per item)
    int32_t nl = 0;
    if (gram_split()) cudaMemcpy(&nl, ws + L.wlist, sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (nl > 0) {
      std::vector<int4> wl((size_t)nl);
      cudaMemcpy(wl.data(), ws + L.wlist + sizeof(int4), sizeof(int4) * nl, cudaMemcpyDeviceToHost);
      for (const int4& e : wl) {
        const int ktp = ((e.z >> 16) + 15) & ~15;
        f += 2.0 * 128.0 * ktp * (double)(a->d + tile::kMaxKpadTC);
      }
    }
    *flops = f;
    return check_launch("tile_executed_flops");
  }
  int32_t nsub = 0;
  cudaMemcpyAsync(&nsub, ws + L.sub, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("tile_executed_flops");
  const int64_t items = L.ntiles + 4 * (int64_t)std::min(nsub, L.max_sub_tiles);
  std::vector<int32_t> kt((size_t)items);
  cudaMemcpy(kt.data(), ws + L.kt, sizeof(int32_t) * items, cudaMemcpyDeviceToHost);
  for (int64_t t = 0; t < items; ++t) {
    const int ktp = (kt[t] + 15) & ~15;
    if (kt[t] > 0 && ktp <= tile::ws_kt_max(x3))
      f += (x3 ? 3.0 : 1.0) * 2.0 * 128.0 * ktp * (double)(a->d + tile::kMaxKpadTC);
  }
  *flops = f;
  return check_launch("tile_executed_flops");
}

}  // extern "C"

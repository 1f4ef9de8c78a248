// Cell-range sharding of one object across the GPUs of a box ("alternative for C5").
//
// Plain point-range sharding (dist.shard_range) leaves every rank touching voxels all over the
// object, so the dense voxel partials must be all-reduced: 2 G^3 floats = 1.07 GB at 512^3, which
// over NVLink costs more than the whole per-rank fused pass at 8 GPUs. Here each point is instead
// routed to the rank that OWNS its voxel:
//
//   1. every rank: key = 3-D Hilbert index of a 64^3 cell grid DERIVED FROM THE VOXEL CODE
//      (cell_a = code_a * 64 / G per axis, integer): every voxel lies in exactly one cell, so an
//      owner of whole cells owns whole voxels, whatever G is; histogram of the keys (2^18 bins);
//   2. all-reduce of the histogram (1 MB, NCCL);
//   3. every rank, identically: cuts = the cell boundaries that split the global count into W
//      balanced ranges along the curve (pf_shard_cuts; rank r owns cells [cut_r, cut_{r+1}));
//   4. pack: the local points grouped by destination rank, each carrying its local index in .w
//      (pf_shard_pack); all-to-all of the packed points (the exchange step);
//   5. the receiver runs the fused path on what it received: its voxels are its own, so the sparse
//      voxel mass over its touched list is final for those voxels; only K + 8 doubles are
//      all-reduced;
//   6. per-point results go back with the reverse all-to-all (pf_shard_pack_results /
//      pf_shard_unpack_results), so each rank ends with the outputs of its own input range in the
//      caller's order — the same contract as range sharding.
// The voxel code used for ownership is computed by the same fp64 expression as the fused path's
// (pf_common.cuh voxel_code), so a point's owner and its partial's voxel always agree.
#include "pf_common.cuh"

namespace pf {
namespace {

constexpr int kCellBits = 6;                        // 64^3 cells
constexpr int kCells = 1 << kCellBits;
constexpr int kBins = 1 << (3 * kCellBits);         // 262144 histogram bins
constexpr int kMaxWorld = 64;

__device__ __forceinline__ uint32_t hilbert3_6(uint32_t x, uint32_t y, uint32_t z) {
  // Skilling's transpose algorithm on a 2^6 grid (as the tile sort's key, pf_tile.cu)
  uint32_t X[3] = {x, y, z};
  const uint32_t M = 1u << (kCellBits - 1);
#pragma unroll
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t Pm = Q - 1;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= Pm;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & Pm;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  X[1] ^= X[0];
  X[2] ^= X[1];
  uint32_t t = 0;
#pragma unroll
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  X[0] ^= t;
  X[1] ^= t;
  X[2] ^= t;
  uint32_t key = 0;
#pragma unroll
  for (int b = kCellBits - 1; b >= 0; --b)
    key = (key << 3) | (((X[0] >> b) & 1u) << 2) | (((X[1] >> b) & 1u) << 1) | ((X[2] >> b) & 1u);
  return key;
}

__global__ void k_shard_keys(const float* __restrict__ p, int64_t n, const double* __restrict__ lo_hi, int g,
                             uint32_t* __restrict__ keys, uint32_t* __restrict__ hist) {
  __shared__ double s_lo[3], s_edge;
  if (threadIdx.x == 0) {
    double lo[3];
    s_edge = voxel_edge(lo_hi, g, lo);
    s_lo[0] = lo[0];
    s_lo[1] = lo[1];
    s_lo[2] = lo[2];
  }
  __syncthreads();
  const double edge = s_edge;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // the fused path's per-axis voxel index (bit-identical expression), then the enclosing cell
    const int cx = voxel_axis(__ldg(p + 3 * i), s_lo[0], edge, g);
    const int cy = voxel_axis(__ldg(p + 3 * i + 1), s_lo[1], edge, g);
    const int cz = voxel_axis(__ldg(p + 3 * i + 2), s_lo[2], edge, g);
    const uint32_t key = hilbert3_6((uint32_t)((int64_t)cx * kCells / g), (uint32_t)((int64_t)cy * kCells / g),
                                    (uint32_t)((int64_t)cz * kCells / g));
    keys[i] = key;
    atomicAdd(hist + key, 1u);
  }
}

// One block of 1024 threads, 256 bins each: block scan of the per-thread sums, then each thread
// walks its bins. Rank r starts at the first bin c whose exclusive prefix reaches
// ceil(r * total / world); ranks whose targets fall on one bin boundary share it (the earlier ones
// get empty ranges).
__global__ void __launch_bounds__(1024) k_shard_cuts(const uint32_t* __restrict__ hist, int world,
                                                     uint32_t* __restrict__ cuts) {
  __shared__ uint64_t s[1024];
  constexpr int kPer = kBins / 1024;
  const int t = threadIdx.x;
  uint64_t mine = 0;
  for (int b = 0; b < kPer; ++b) mine += hist[t * kPer + b];
  s[t] = mine;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan
    const uint64_t v = t >= o ? s[t - o] : 0ull;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  const uint64_t total = s[1023];
  if (t == 0) {  // targets past the last non-empty bin start at the end
    cuts[0] = 0u;
    for (int r = 1; r <= world; ++r) cuts[r] = (uint32_t)kBins;
  }
  __syncthreads();
  uint64_t prefix = s[t] - mine;  // prefix(first bin of this thread)
  uint32_t prev = t == 0 ? 0u : hist[t * kPer - 1];
  for (int b = 0; b < kPer; ++b) {
    const uint32_t bin = (uint32_t)(t * kPer + b);
    const uint32_t h = hist[bin];
    for (int r = 1; r < world; ++r) {
      const uint64_t target = (total * (uint64_t)r + (uint64_t)world - 1) / (uint64_t)world;
      if (prefix >= target && (bin == 0 || prefix - prev < target)) cuts[r] = bin;
    }
    prefix += h;
    prev = h;
  }
}

__device__ __forceinline__ int owner_of(uint32_t key, const uint32_t* cuts, int world) {
  int r = 0;
  for (int q = 1; q < world; ++q) r += key >= cuts[q] ? 1 : 0;  // cuts are non-decreasing
  return r;
}

// Grid-stride over chunks of blockDim points. Per chunk: warp-aggregated shared counters per
// destination (__match_any_sync), one global reservation per (block, destination), then the
// writes — no per-point global atomics on the W cursors.
template <bool kScatter>
__global__ void __launch_bounds__(256) k_shard_route(const float* __restrict__ p, int64_t n,
                                                     const uint32_t* __restrict__ keys,
                                                     const uint32_t* __restrict__ cuts, int world,
                                                     int32_t* __restrict__ cursor, float4* __restrict__ send) {
  __shared__ uint32_t s_cut[kMaxWorld + 1];
  __shared__ int32_t s_cnt[kMaxWorld], s_base[kMaxWorld];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int q = tid; q <= world; q += blockDim.x) s_cut[q] = cuts[q];
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + tid;
    const bool valid = i < n;
    if (tid < world) s_cnt[tid] = 0;
    __syncthreads();
    const int r = valid ? owner_of(keys[i], s_cut, world) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    const int leader = __ffs(peers) - 1;
    int off = 0;
    if (valid && lane == leader) off = atomicAdd(&s_cnt[r], __popc(peers));
    off = __shfl_sync(0xffffffffu, off, leader) + __popc(peers & ((1u << lane) - 1u));
    __syncthreads();
    if (tid < world) {
      const int32_t c = s_cnt[tid];
      s_base[tid] = c ? atomicAdd(cursor + tid, c) : 0;
    }
    __syncthreads();
    if (kScatter && valid)
      send[s_base[r] + off] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2),
                                          __int_as_float((int32_t)i));
    __syncthreads();
  }
}

__global__ void k_shard_offsets(const int32_t* __restrict__ counts, int world, int32_t* __restrict__ cursor) {
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int q = 0; q < world; ++q) {
      cursor[q] = acc;
      acc += counts[q];
    }
  }
}

// received float4 points -> packed (n,3) f32 for the fused path
__global__ void k_shard_xyz(const float4* __restrict__ recv, int64_t n, float* __restrict__ xyz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 q = recv[i];
    xyz[3 * i] = q.x;
    xyz[3 * i + 1] = q.y;
    xyz[3 * i + 2] = q.z;
  }
}

// one int32 row per point: [props (P f32 bits) | count | code | mask words]
__global__ void k_shard_pack_results(int64_t n, int p, int nwords, const float* __restrict__ props,
                                     const int32_t* __restrict__ counts, const int32_t* __restrict__ codes,
                                     const int32_t* __restrict__ mask, int32_t* __restrict__ rows) {
  const int w = p + 2 + nwords;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t* r = rows + i * w;
    for (int c = 0; c < p; ++c) r[c] = __float_as_int(props[i * p + c]);
    r[p] = counts[i];
    r[p + 1] = codes[i];
    for (int c = 0; c < nwords; ++c) r[p + 2 + c] = mask[i * nwords + c];
  }
}

// row j of the returned block belongs to the local point whose index the sent float4 j carried
__global__ void k_shard_unpack_results(int64_t n, int p, int nwords, const int32_t* __restrict__ rows,
                                       const float4* __restrict__ sent, float* __restrict__ props,
                                       int32_t* __restrict__ counts, int32_t* __restrict__ codes,
                                       int32_t* __restrict__ mask) {
  const int w = p + 2 + nwords;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = __float_as_int(sent[j].w);
    const int32_t* r = rows + j * w;
    for (int c = 0; c < p; ++c) props[i * p + c] = __int_as_float(r[c]);
    counts[i] = r[p];
    codes[i] = r[p + 1];
    for (int c = 0; c < nwords; ++c) mask[i * nwords + c] = r[p + 2 + c];
  }
}

// ---- fixed-capacity exchange (no host synchronisation) ---------------------------------------------
// send / recv blocks: W x (C + 1) float4; row 0 of block o = {count (int bits), flags, 0, 0}, rows
// 1.. the points for owner o. Unused rows are NaN points: the fused path treats a NaN point as a
// padding slot (invisible, voxel code -1, no voxel / partial contribution), so the receiver runs a
// fixed W*C-point pass whose size the host knows without reading the counts back.
__global__ void __launch_bounds__(256) k_shard_route_padded(const float* __restrict__ p, int64_t n,
                                                            const uint32_t* __restrict__ keys,
                                                            const uint32_t* __restrict__ cuts, int world, int cap,
                                                            int32_t* __restrict__ cursor, float4* __restrict__ send,
                                                            int32_t* __restrict__ flags) {
  __shared__ uint32_t s_cut[kMaxWorld + 1];
  __shared__ int32_t s_cnt[kMaxWorld], s_base[kMaxWorld];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int q = tid; q <= world; q += blockDim.x) s_cut[q] = cuts[q];
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + tid;
    const bool valid = i < n;
    if (tid < world) s_cnt[tid] = 0;
    __syncthreads();
    const int r = valid ? owner_of(keys[i], s_cut, world) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, r);
    const int leader = __ffs(peers) - 1;
    int off = 0;
    if (valid && lane == leader) off = atomicAdd(&s_cnt[r], __popc(peers));
    off = __shfl_sync(0xffffffffu, off, leader) + __popc(peers & ((1u << lane) - 1u));
    __syncthreads();
    if (tid < world) {
      const int32_t c = s_cnt[tid];
      s_base[tid] = c ? atomicAdd(cursor + tid, c) : 0;
    }
    __syncthreads();
    if (valid) {
      const int slot = s_base[r] + off;
      if (slot < cap)
        send[(int64_t)r * (cap + 1) + 1 + slot] = make_float4(__ldg(p + 3 * i), __ldg(p + 3 * i + 1),
                                                              __ldg(p + 3 * i + 2), __int_as_float((int32_t)i));
      else
        atomicOr(flags, 1);  // more points for one owner than the capacity: dropped, flagged
    }
    __syncthreads();
  }
}

// per-block header (count, flags) and NaN padding of the unused rows
__global__ void k_shard_pad_finish(float4* __restrict__ send, const int32_t* __restrict__ cursor, int world,
                                   int cap, const int32_t* __restrict__ flags) {
  const float nan = __int_as_float(0x7fc00000);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)world * (cap + 1);
       e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / (cap + 1)), row = (int)(e % (cap + 1));
    const int cnt = min(cursor[o], cap);
    if (row == 0) send[e] = make_float4(__int_as_float(cnt), __int_as_float(*flags), 0.f, 0.f);
    else if (row - 1 >= cnt) send[e] = make_float4(nan, nan, nan, __int_as_float(-1));
  }
}

// received blocks -> (W*C, 3) points in slot order (NaN rows stay NaN: padding)
__global__ void k_shard_unpad(const float4* __restrict__ recv, int world, int cap, float* __restrict__ xyz) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)world * cap;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(e / cap), c = (int)(e % cap);
    const float4 q = recv[(int64_t)s * (cap + 1) + 1 + c];
    xyz[3 * e] = q.x;
    xyz[3 * e + 1] = q.y;
    xyz[3 * e + 2] = q.z;
  }
}

// the owner's result rows come back in slot order: row (o, c) belongs to the local point whose
// index the sent float4 (o, c) carried, for c < the block's count
__global__ void k_shard_unpack_results_padded(int world, int cap, int p, int nwords, const int32_t* __restrict__ rows,
                                              const float4* __restrict__ sent, float* __restrict__ props,
                                              int32_t* __restrict__ counts, int32_t* __restrict__ codes,
                                              int32_t* __restrict__ mask) {
  const int w = p + 2 + nwords;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)world * cap;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / cap), c = (int)(e % cap);
    if (c >= __float_as_int(sent[(int64_t)o * (cap + 1)].x)) continue;
    const int64_t i = __float_as_int(sent[(int64_t)o * (cap + 1) + 1 + c].w);
    const int32_t* r = rows + e * w;
    for (int q = 0; q < p; ++q) props[i * p + q] = __int_as_float(r[q]);
    counts[i] = r[p];
    codes[i] = r[p + 1];
    for (int q = 0; q < nwords; ++q) mask[i * nwords + q] = r[p + 2 + q];
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" {

int32_t pf_shard_bins(void) { return kBins; }

int pf_shard_keys(const float* points, int64_t n, const double* lo_hi, int32_t g, uint32_t* keys, uint32_t* hist,
                  void* stream) {
  if (g < 1) return set_error(PF_ERR_VALUE, "voxel grid side must be >= 1");
  if (n < 0) return set_error(PF_ERR_VALUE, "negative point count");
  if (n == 0) return PF_OK;
  if (!points || !lo_hi || !keys || !hist) return set_error(PF_ERR_VALUE, "shard_keys: null buffer");
  k_shard_keys<<<grid_for(n, 256), 256, 0, S(stream)>>>(points, n, lo_hi, g, keys, hist);
  return check_launch("shard_keys");
}

int pf_shard_cuts(const uint32_t* hist, int32_t world, uint32_t* cuts, void* stream) {
  if (world < 1 || world > kMaxWorld) return set_error(PF_ERR_VALUE, "world size must be in [1, 64]");
  if (!hist || !cuts) return set_error(PF_ERR_VALUE, "shard_cuts: null buffer");
  k_shard_cuts<<<1, 1024, 0, S(stream)>>>(hist, world, cuts);
  return check_launch("shard_cuts");
}

int pf_shard_pack(const float* points, int64_t n, const uint32_t* keys, const uint32_t* cuts, int32_t world,
                  int32_t* counts, int32_t* cursor, void* send, void* stream) {
  if (world < 1 || world > kMaxWorld) return set_error(PF_ERR_VALUE, "world size must be in [1, 64]");
  if (n < 0 || n > INT32_MAX) return set_error(PF_ERR_VALUE, "point count must be in [0, 2^31)");
  if (!counts || !cursor || !cuts) return set_error(PF_ERR_VALUE, "shard_pack: null buffer");
  cudaMemsetAsync(counts, 0, sizeof(int32_t) * world, S(stream));
  if (n > 0) {
    if (!points || !keys || !send) return set_error(PF_ERR_VALUE, "shard_pack: null buffer");
    k_shard_route<false><<<grid_for(n, 256), 256, 0, S(stream)>>>(nullptr, n, keys, cuts, world, counts, nullptr);
    if (int rc = check_launch("shard_count")) return rc;
  }
  k_shard_offsets<<<1, 32, 0, S(stream)>>>(counts, world, cursor);
  if (int rc = check_launch("shard_offsets")) return rc;
  if (n == 0) return PF_OK;
  k_shard_route<true><<<grid_for(n, 256), 256, 0, S(stream)>>>(points, n, keys, cuts, world, cursor,
                                                               reinterpret_cast<float4*>(send));
  return check_launch("shard_scatter");
}

int pf_shard_xyz(const void* recv, int64_t n, float* xyz, void* stream) {
  if (n <= 0) return n < 0 ? set_error(PF_ERR_VALUE, "negative point count") : PF_OK;
  if (!recv || !xyz) return set_error(PF_ERR_VALUE, "shard_xyz: null buffer");
  k_shard_xyz<<<grid_for(n, 256), 256, 0, S(stream)>>>(reinterpret_cast<const float4*>(recv), n, xyz);
  return check_launch("shard_xyz");
}

int pf_shard_pack_results(int64_t n, int32_t p, int32_t nwords, const float* props, const int32_t* counts,
                          const int32_t* codes, const int32_t* mask, int32_t* rows, void* stream) {
  if (n <= 0) return n < 0 ? set_error(PF_ERR_VALUE, "negative point count") : PF_OK;
  if (!props || !counts || !codes || !mask || !rows) return set_error(PF_ERR_VALUE, "shard_pack_results: null buffer");
  k_shard_pack_results<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, p, nwords, props, counts, codes, mask, rows);
  return check_launch("shard_pack_results");
}

int pf_shard_unpack_results(int64_t n, int32_t p, int32_t nwords, const int32_t* rows, const void* sent,
                            float* props, int32_t* counts, int32_t* codes, int32_t* mask, void* stream) {
  if (n <= 0) return n < 0 ? set_error(PF_ERR_VALUE, "negative point count") : PF_OK;
  if (!rows || !sent || !props || !counts || !codes || !mask)
    return set_error(PF_ERR_VALUE, "shard_unpack_results: null buffer");
  k_shard_unpack_results<<<grid_for(n, 256), 256, 0, S(stream)>>>(n, p, nwords, rows,
                                                                  reinterpret_cast<const float4*>(sent), props,
                                                                  counts, codes, mask);
  return check_launch("shard_unpack_results");
}

int pf_shard_pack_padded(const float* points, int64_t n, const uint32_t* keys, const uint32_t* cuts, int32_t world,
                         int32_t capacity, int32_t* cursor, void* send, int32_t* flags, void* stream) {
  if (world < 1 || world > kMaxWorld) return set_error(PF_ERR_VALUE, "world size must be in [1, 64]");
  if (n < 0 || n > INT32_MAX) return set_error(PF_ERR_VALUE, "point count must be in [0, 2^31)");
  if (capacity < 1) return set_error(PF_ERR_VALUE, "capacity must be >= 1");
  if (!cursor || !cuts || !send || !flags) return set_error(PF_ERR_VALUE, "shard_pack_padded: null buffer");
  cudaMemsetAsync(cursor, 0, sizeof(int32_t) * world, S(stream));
  cudaMemsetAsync(flags, 0, sizeof(int32_t), S(stream));
  if (n > 0) {
    if (!points || !keys) return set_error(PF_ERR_VALUE, "shard_pack_padded: null buffer");
    k_shard_route_padded<<<grid_for(n, 256), 256, 0, S(stream)>>>(points, n, keys, cuts, world, capacity, cursor,
                                                                 reinterpret_cast<float4*>(send), flags);
    if (int rc = check_launch("shard_route_padded")) return rc;
  }
  k_shard_pad_finish<<<grid_for((int64_t)world * (capacity + 1), 256), 256, 0, S(stream)>>>(
      reinterpret_cast<float4*>(send), cursor, world, capacity, flags);
  return check_launch("shard_pad_finish");
}

int pf_shard_unpad(const void* recv, int32_t world, int32_t capacity, float* xyz, void* stream) {
  if (world < 1 || world > kMaxWorld || capacity < 1) return set_error(PF_ERR_VALUE, "shard_unpad: bad shape");
  if (!recv || !xyz) return set_error(PF_ERR_VALUE, "shard_unpad: null buffer");
  k_shard_unpad<<<grid_for((int64_t)world * capacity, 256), 256, 0, S(stream)>>>(reinterpret_cast<const float4*>(recv),
                                                                                world, capacity, xyz);
  return check_launch("shard_unpad");
}

int pf_shard_unpack_results_padded(int32_t world, int32_t capacity, int32_t p, int32_t nwords, const int32_t* rows,
                                   const void* sent, float* props, int32_t* counts, int32_t* codes, int32_t* mask,
                                   void* stream) {
  if (world < 1 || world > kMaxWorld || capacity < 1) return set_error(PF_ERR_VALUE, "unpack_results_padded: bad shape");
  if (!rows || !sent || !props || !counts || !codes || !mask)
    return set_error(PF_ERR_VALUE, "shard_unpack_results_padded: null buffer");
  k_shard_unpack_results_padded<<<grid_for((int64_t)world * capacity, 256), 256, 0, S(stream)>>>(
      world, capacity, p, nwords, rows, reinterpret_cast<const float4*>(sent), props, counts, codes, mask);
  return check_launch("shard_unpack_results_padded");
}

}  // extern "C"

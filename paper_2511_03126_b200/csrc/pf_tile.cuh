// Shared declarations of the tensor-core tile path (pf_tile.cu, pf_tile_ws.cu) and its host
// orchestration.
//
// Data flow (all per-point intermediates live in SORTED order, so every pass over them is
// coalesced; the original order is touched once, by a gather in k_unsort):
//   k_sort_scatter : spts[j] = {x, y, z, bits(i)}, inv[i] = j          (j = Hilbert-sorted slot)
//   k_tile_prep    : srec[j].{mask, count, code}, per-tile tap windows
//   k_tile_ws      : srec[j].prop, voxel + integrate partials
//   k_unsort       : outputs[i] <- srec[inv[i]]  (one 32-byte sector read per point)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/propfield_b200.h"

namespace pf {
namespace tile {

constexpr int kTile = 128;             // points per tile = tcgen05 M
constexpr int kMaxViewsTC = 64;        // views supported by the tile path (2 bitset words)
constexpr int kMaxKpadTC = 128;        // padded materials (MMA N of the S chunk pair)
constexpr int kSortBitsMax = 8;        // Hilbert curve over a 2^bits cube grid over the bbox:
constexpr int kSortBinsMax = 1 << (3 * kSortBitsMax);  // 7 bits (128^3), 8 bits (256^3) from 4M points
inline int sort_bits_for(int64_t n) { return n >= (int64_t(1) << 22) ? 8 : 7; }

struct ViewF {
  float R[9];
  float t[3];
  float fx, fy, cx, cy;
  float ru, rv;  // Wf / W, Hf / H
  float tmax;
  int H, W, Hf, Wf;
  int32_t cell_base;
  int64_t depth_off;
};

struct TapF {
  int x0, y0, dx, dy;
  float wx, wy;
};

// one point's record in sorted order (32 bytes = one DRAM sector)
struct __align__(32) SRec {
  uint32_t m0, m1;  // visibility bitset (views 0-31, 32-63)
  int32_t count;    // visible views
  int32_t code;     // voxel code
  float prop[4];    // regressed properties (P <= 4)
};

struct TileParams {
  const float4* spts;   // sorted points, .w = original index (int bits)
  const int32_t* inv;   // original index -> sorted slot
  SRec* srec;           // sorted per-point records
  int64_t n;
  const pf_view_t* views;
  int nv, nwords, d;
  const float* depth;
  const void* fmap;     // bf16 packed maps (x3: the bf16 high parts of the f32 maps)
  const uint16_t* Gbf;  // (cells, kpadg) bf16 (x3: high parts)
  // x3 (f32 maps): every f32 operand is split hi + lo into bf16 and each MMA k-step issues
  // hi.hi + hi.lo + lo.hi (fp32-accurate to ~2^-16); kt_max = taps per work item held by one A buffer
  const uint16_t* fmap_lo;
  const uint16_t* Gbf_lo;
  int32_t x3, kt_max;
  int kpadg, k, p, density_col;
  const float* values;
  const float* mid_theta;
  float inv_temp;
  double eps;
  int grid;
  int64_t cells3;
  const double* lo_hi;
  uint32_t* mask_bits;   // outputs in original order (k_unsort)
  int32_t* counts;
  int32_t* codes;
  float* props;
  float* grid_partials;  // nullptr: skip voxels
  int32_t* vox_list;     // optional touched-voxel list (first point of a voxel appends its code)
  int32_t* vox_count;
  float* features;       // optional validation outputs, original order
  float* sims;
  float* weights;
  int32_t* status;
  uint2* tile_desc;
  int32_t* tile_kt;
  ViewF* viewf;   // per-view fp32 camera (k_view_setup)
  float4* vbound; // per-view constant error bounds over the bbox (k_view_setup)
  double* vox;    // voxel domain (k_view_setup): lo (3), edge (fp64), then lo (3) and 1/edge as f32 bits
  int32_t* ovf_list;
  int32_t* ovf_count;
  // overflow tiles (more taps than one A buffer) are re-run as 4 sub-tiles of 32 rows: work items
  // ntiles + 4 b + q (b < min(*sub_count, max_sub_tiles)) cover rows 32q.. of tile sub_tiles[b]
  int32_t* sub_tiles;
  int32_t* sub_count;
  int32_t max_sub_tiles;
  // Gram path (pf_gram.cu): work items are the 512-row tiles (ids < ntiles), the 128-row tiles
  // (ids ntiles + t128: the level-1 items of overflowing tiles) and 32-row splits of overflowing
  // 128-row tiles (ids ntiles + 4 max_sub_tiles + 4 c + q, c < min(*sub2_count, max_sub2), rows 32 q
  // .. of the 128-row tile with item id sub2_items[c]). k_tile_ws uses tr = 128, sub1_rows = 32
  // (level-1 items ntiles + 4 b + q: rows 32 q .. of tile sub_tiles[b]).
  int32_t tr, sub1_rows;
  int32_t* sub2_items;
  int32_t* sub2_count;
  int32_t max_sub2;
  unsigned long long* dbg;  // optional counters (PF_WS_DEBUG)
  int32_t ablate;           // Gram kernel timing experiments only (PF_GRAM_ABLATE bits; results invalid)
  int32_t deterministic;    // PF_FUSE_DETERMINISTIC: stable radix sort (run-to-run identical tiles)
  uint32_t* trace;          // optional per-tile role timestamps (PF_WS_DEBUG + PF_WS_TRACE=<file>)
  double* partials;
  // Gram path: compact list of the work items that run in the tile kernel ({item, first row,
  // rows | taps << 16, 0}, k_collect_work) and its length
  int4* work;
  int32_t* work_count;
  int4* work_raw;  // k_collect_work's output (arbitrary order); k_sort_work -> work
  // Gram path: the 128- and 32-row items (split tiles) run in k_tile_ws from this list instead
  // (same entry format); nullptr: k_tile_ws walks its own tile / sub-tile items
  int4* wlist;
  int32_t* wcount;
  const float* tbound;  // max_k |t_k| (run_text_bound, per object): bounds the softmax exponents
  // Gram path: box of every 128-row tile ({lo.xyz, -}, {hi.xyz, -}; k_tile_prep): the builders'
  // expansion centre of an item
  float4* tbox;
  unsigned long long* ctatime;  // optional per-CTA start / end times of the Gram kernel (PF_GRAM_CTATIME)
};

struct TileLayout {
  int64_t ntiles;
  int32_t max_sub_tiles, max_sub2;
  size_t keys, hist, totals, keys_out, idx, idx_out, sort_tmp, inv, spts, srec, desc, kt, ovf, sub, sub2, work, work_raw, wlist, tbox, gbf, textbf, viewf, vbound, vox, tbound, glo, fhi, flo, textlo,
      bytes;
};

TileLayout tile_layout(int64_t n, int nv, int64_t cells, int kpadg, int d = 0, bool x3 = false, int tr = 128);
// x3 operands of f32 maps: hi = bf16(x), lo = bf16(x - hi), for the maps and the G table
int run_split_f32(const float* src, int64_t rows, int cols, int src_ld, int dst_ld, uint16_t* hi, uint16_t* lo,
                  cudaStream_t st);
// fork (optional): called before the point sort is enqueued; it enqueues the per-object tables
// (pf_fuse_prepare) on a forked stream and returns the event the tensor-core kernels wait on (null:
// nothing to wait for), so the tables are built while the points are sorted
struct ForkHook {
  cudaEvent_t (*fn)(void* ctx, cudaStream_t st, int* rc) = nullptr;
  void* ctx = nullptr;
  cudaEvent_t depth_ready = nullptr;  // staged inputs (pf_fuse_args_t): waited on before the prep
  cudaEvent_t fmap_ready = nullptr;   // ... and before the tensor-core kernel
};
int run_tile_path(TileParams P, const TileLayout& L, unsigned char* ws, const float* points,
                  int64_t n, cudaStream_t st, ForkHook fork = ForkHook{}, cudaEvent_t* joined = nullptr);
int run_unsort(const TileParams& P, cudaStream_t st);
int run_tile_ws(const TileParams& P, cudaStream_t st);
// Gram formulation (pf_gram.cu): bf16 maps, no mean-feature output
int run_tile_gram(const TileParams& P, cudaStream_t st);
constexpr int kGramTile = 512;   // rows of a level-0 tile of the Gram path
constexpr int kGramKt = 192;     // taps per work item held by the Gram kernel
int run_g_bf16(const float* G, int64_t cells, int kpad, int kpadg, uint16_t* Gbf, cudaStream_t st);
int run_gproj_tc(const void* fmap, int64_t cells, int d, const float* text, int k, int kpadg, int kpad,
                 uint16_t* Gbf, float* G32, uint16_t* textbf, cudaStream_t st);
int ws_kt_max(bool x3 = false);
int run_text_bound(const float* text, int k, int d, float* out, cudaStream_t st);
int run_gproj_tc_x3(const uint16_t* fhi, const uint16_t* flo, int64_t cells, int d, const float* text, int k,
                    int kpadg, int kpad, uint16_t* Gbf, uint16_t* Gbf_lo, float* G32, uint16_t* text_hi,
                    uint16_t* text_lo, cudaStream_t st);
// add_block_bases = false leaves hist[i] block-local (exclusive within its 4096-bin block) and
// totals[b] the exclusive base of block b: the consumer adds totals[i >> 12] itself
int run_bucket_scan(uint32_t* hist, uint32_t* totals, int64_t nbins, cudaStream_t st, bool add_block_bases = true);
// Hilbert order of the points for the SIMT path: order[t] = index of the t-th point along the curve
// (7-bit key over the domain lo_hi), and *len = n (the kernel's list length). ws: point_order_bytes.
size_t point_order_bytes(int64_t n);
int run_point_order(const float* points, int64_t n, const double* lo_hi, unsigned char* ws, int32_t* order,
                    int32_t* len, cudaStream_t st);
constexpr int kSubRows = 32;  // rows of a sub-tile
constexpr int kSubPerTile = kTile / kSubRows;

}  // namespace tile
}  // namespace pf

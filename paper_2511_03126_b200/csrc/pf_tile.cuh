// Shared declarations of the tensor-core tile path (pf_tile.cu) and its host orchestration.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/propfield_b200.h"

namespace pf {
namespace tile {

constexpr int kTile = 128;             // points per tile = tcgen05 M
constexpr int kKtMax = 192;            // taps per tile held in shared memory
constexpr int kMaxViewsTC = 64;        // views supported by the tile path (2 bitset words)
constexpr int kMaxKpadTC = 128;        // padded materials (MMA N of the S chunk; B tile <= 2 halves)
constexpr int kRedStride = kMaxKpadTC + 1;
constexpr int kSortBits = 7;           // Morton grid 128^3 over the bbox
constexpr int kSortCells = 1 << kSortBits;
constexpr int kSortBins = 1 << (3 * kSortBits);

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

struct TileParams {
  const float4* spts;   // sorted points
  const int32_t* perm;  // sorted slot -> original index
  int64_t n;
  const pf_view_t* views;
  int nv, nwords, d;
  const float* depth;
  const void* fmap;     // bf16 packed maps
  const uint16_t* Gbf;  // (cells, kpadg) bf16
  int kpadg, k, p, density_col;
  const float* values;
  const float* mid_theta;
  float inv_temp;
  double eps;
  int grid;
  int64_t cells3;
  const double* lo_hi;
  uint32_t* mask_bits;
  int32_t* counts;
  int32_t* codes;
  float* props;
  float* grid_partials;  // nullptr: skip voxels
  float* features;
  float* sims;
  float* weights;
  int32_t* status;
  uint2* tile_desc;
  int32_t* tile_kt;
  float* tile_part;
  ViewF* viewf;   // per-view fp32 camera (k_view_setup)
  float4* vbound; // per-view constant error bounds over the bbox (k_view_setup)
  int32_t* ovf_list;
  int32_t* ovf_count;
  unsigned long long* dbg;  // optional per-CTA wait-cycle counters (PF_WS_DEBUG)
  double* partials;
  uint32_t tmem_cols;
};

struct TileLayout {
  int64_t ntiles;
  size_t keys, hist, totals, perm, spts, desc, kt, part, ovf, gbf, viewf, vbound, bytes;
};

TileLayout tile_layout(int64_t n, int nv, int64_t cells, int kpadg);
size_t tile_smem_bytes();
int run_tile_path(TileParams P, const TileLayout& L, unsigned char* ws, const float* points,
                  int64_t n, int64_t cells, const float* G, int kpad, int hf, int wf, cudaStream_t st);
int run_tile_ws(const TileParams& P, int hf, int wf, int nv, cudaStream_t st);
int run_g_bf16(const float* G, int64_t cells, int kpad, int kpadg, uint16_t* Gbf, cudaStream_t st);
int run_gproj_tc(const void* fmap, int64_t cells, int d, const float* text, int k, int kpadg, int kpad,
                 uint16_t* Gbf, float* G32, cudaStream_t st);

}  // namespace tile
}  // namespace pf

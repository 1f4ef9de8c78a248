/*
 * propfield_b200.h — C ABI of the B200-native fusion + property-query path.
 *
 * Drop-in boundary for the reference's hot path. Each entry point below names the
 * reference interface it replaces (file:line under /root/reference/pkg/src/propfield/). The Python
 * package paper_2511_03126_b200 binds these symbols with ctypes (INTEGRATION.md shows the binding);
 * any other FFI (cffi, a C++ caller, cgo) can bind them the same way.
 *
 * Conventions (all entry points):
 *   - Every pointer argument is a DEVICE pointer unless its name ends in `_host`.
 *   - The caller allocates every buffer (outputs and workspace). The library never allocates or
 *     frees caller memory and keeps no global device state; `pf_*_workspace_bytes` size workspaces.
 *   - Calls are stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream) and are
 *     re-entrant for distinct output buffers. Nothing synchronises unless documented.
 *   - Return value: PF_OK (0) or a PF_ERR_* status. `pf_last_error()` returns a thread-local
 *     message for the last failing call on this thread. The Python binding maps statuses to the
 *     reference's exception classes (errors.py:4-37): VALUE -> ValueError, STRUCTURE ->
 *     BundleStructureError, MATERIAL -> MaterialError, CUDA -> CudaError.
 *   - There is no CPU fallback and no backend switch: without a CUDA device every call fails
 *     with PF_ERR_CUDA.
 */
#ifndef PROPFIELD_B200_H
#define PROPFIELD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 1

enum pf_status {
  PF_OK = 0,
  PF_ERR_VALUE = 1,     /* bad scalar argument, e.g. temperature <= 0 (grounding.py:170-171) */
  PF_ERR_STRUCTURE = 2, /* inconsistent shapes / unsupported layout (bundle.py:45-55,105-116)   */
  PF_ERR_MATERIAL = 3,  /* NaN similarity / missing property (grounding.py:69-72,173-174)       */
  PF_ERR_CUDA = 4,      /* CUDA runtime failure (no reference twin)                             */
  PF_ERR_LOAD = 5       /* missing / unreadable file (BundleLoadError, tensorio.py:44-47)       */
};

enum pf_dtype { PF_F32 = 0, PF_BF16 = 1, PF_F64 = 2 };

/* One posed view, packed for the device (bundle.py:35-116: CameraPose, Intrinsics, ViewRecord).
 * R is the row-major world->camera rotation, x_cam = R x_world + t. `depth_offset` / `fmap_offset`
 * are ELEMENT offsets of this view's (H,W) f32 depth map and (Hf,Wf,D) channel-last feature map
 * inside the packed buffers passed alongside. 160 bytes, 8-byte aligned. */
typedef struct pf_view {
  double R[9];
  double t[3];
  double fx, fy, cx, cy;
  int64_t depth_offset;
  int64_t fmap_offset;
  int32_t H, W;
  int32_t Hf, Wf;
} pf_view_t;

const char* pf_last_error(void);
int pf_abi_version(void);
/* Number of this library's kernel launches issued by the calling thread since load (for bench). */
uint64_t pf_launch_count(void);

/* ---------------------------------------------------------------------------------------------
 * Operator level: the `propfield.kernels` registry (kernels/__init__.py:21-28). fp64, bit-exact
 * with the reference's numpy twins (same operation order, no FMA contraction).
 * ------------------------------------------------------------------------------------------- */

/* kernels.visible_in_view (numpy_impl.py:14-40, numba_impl.py:15-32). out: (n,) uint8 0/1. */
int pf_visible_in_view(const double* u, const double* v, const double* z, int64_t n,
                       const float* depth, int32_t h, int32_t w, double eps, uint8_t* out,
                       void* stream);

/* kernels.bilinear_gather (numpy_impl.py:43-66). fmap (hf,wf,d) f32|bf16 channel-last;
 * out (m,d) f64. */
int pf_bilinear_gather(const void* fmap, int32_t fmap_dtype, int32_t hf, int32_t wf, int32_t d,
                       const double* fu, const double* fv, int64_t m, double* out, void* stream);

/* kernels.accumulate_features (numpy_impl.py:69-77): accum[rows] += sample; counts[rows] += 1.
 * MUTATES accum (n_rows,d) f64 and counts (n_rows,) int64 in place. Rows must be unique. */
int pf_accumulate_features(const void* fmap, int32_t fmap_dtype, int32_t hf, int32_t wf, int32_t d,
                           const double* fu, const double* fv, const int64_t* rows, int64_t m,
                           double* accum, int64_t* counts, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Function level: geometry / fusion / grounding (the entry points pipeline.py:224-232,275-281
 * calls). fp64, matching the reference to float rounding.
 * ------------------------------------------------------------------------------------------- */

/* geometry.project_points (geometry.py:46-59): points (n,3) f64 -> uv (n,2) f64, z (n,) f64. */
int pf_project_points(const double* points, int64_t n, const pf_view_t* view_host, double* uv,
                      double* z, void* stream);

/* geometry.visibility_mask (geometry.py:89-103). points (n,3) in `points_dtype` (F32 or F64);
 * views (nviews) device array; depth packed f32. mask (n,nviews) uint8 0/1 row-major. */
int pf_visibility_mask(const void* points, int32_t points_dtype, int64_t n, const pf_view_t* views,
                       int32_t nviews, const float* depth, double eps, uint8_t* mask,
                       void* stream);

/* fusion.aggregate_geometric_features (fusion.py:65-93). visibility (n,nviews) uint8; features
 * (n,d) f64 (mean over visible views, zero rows for featureless points); counts (n,) int64.
 * Bit-exact with the reference (per-view fp64 accumulation in view order). */
int pf_aggregate_features(const void* points, int32_t points_dtype, int64_t n,
                          const pf_view_t* views, int32_t nviews, const void* fmap,
                          int32_t fmap_dtype, int32_t d, const uint8_t* visibility,
                          double* features, int64_t* counts, void* stream);

/* grounding.material_similarity (grounding.py:158-165): out (s,k) = f (s,d) @ text (k,d)^T, f64. */
int pf_material_similarity(const double* features, int64_t s, int32_t d, const double* text,
                           int32_t k, double* out, void* stream);

/* grounding.softmax_weights (grounding.py:168-178). temperature <= 0 -> PF_ERR_VALUE. A NaN
 * similarity sets *nan_flag (device int32, caller-zeroed) to 1; the binding raises MaterialError.
 * Rows flagged in `row_valid` (uint8, may be NULL = all valid) == 0 produce all-zero rows
 * (pipeline.py:279-280 featureless convention). */
int pf_softmax_weights(const double* sims, int64_t s, int32_t k, double temperature,
                       const uint8_t* row_valid, double* weights, int32_t* nan_flag, void* stream);

/* grounding.regress_with_weights (grounding.py:198-202): out (s,p) = w (s,k) @ y (k,p), f64. */
int pf_regress_with_weights(const double* weights, int64_t s, int32_t k, const double* values,
                            int32_t p, double* out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Voxel-grid mass (BASELINE-defined; indexing convention of sampling.py:110-123)
 * and integrate_mass partials (integrate.py:124-155).
 * ------------------------------------------------------------------------------------------- */

/* Per-axis bbox of points (n,3) f32 -> lo_hi[6] f64 = {lo_x,lo_y,lo_z,hi_x,hi_y,hi_z}. Exact. */
int pf_bbox(const float* points, int64_t n, double* lo_hi, void* stream);

/* Voxel codes: edge = max(hi-lo)/g, cell = clip(floor((p-lo)/edge),0,g-1) in fp64,
 * code = (cx*g+cy)*g+cz (int32; g <= 1290). Bit-exact. domain = lo_hi as from pf_bbox. */
int pf_voxel_codes(const float* points, int64_t n, const double* lo_hi, int32_t g, int32_t* codes,
                   void* stream);

/* Dense voxel partials: grid (2*g^3) f32 = [sum rho | count], caller-zeroed; add each point. */
int pf_voxel_accumulate(const int32_t* codes, const float* rho, int64_t n, int32_t g, float* grid,
                        void* stream);

/* mass = edge^3 * sum_{count>0} sum/count over the (allreduced) grid. `out` is a caller-zeroed
 * device double[2] = {mass_kg, occupied_voxels}; lo_hi as above (edge recomputed identically). */
int pf_voxel_mass(const float* grid, int32_t g, const double* lo_hi, double* out, void* stream);
/* The same mass from the touched-voxel list of pf_fuse_query (one GPU: no dense scan); zeroes the
 * listed grid entries, leaving the grid clean for the next object. capacity = n (the list holds 2n). */
int pf_voxel_mass_sparse(float* grid, int32_t g, const int32_t* list, const int32_t* count, int64_t capacity,
                         const double* lo_hi, double* out, void* stream);

/* integrate.characteristic_length (integrate.py:72-95), device part: for every point of (n,3) f32,
 * the squared distance to its (k+1)-th nearest point, self included (cKDTree.query(p, k+1)[:, k]),
 * exact, in fp64; *dk2_sum (device f64) = their sum. dk_sorted (nullable, device f32 (n)) receives
 * the distances in the library's internal bucket order. Workspace: pf_knn_workspace_bytes(n). */
uint64_t pf_knn_workspace_bytes(int64_t n);
int pf_knn_kth_distance(const float* points, int64_t n, int32_t k, double* dk2_sum, float* dk_sorted,
                        void* workspace, void* stream);

/* integrate_mass partials (integrate.py:124-155) from a probability matrix: weights (n,k) f64
 * row-major, positions (n,3) f32, normals (n,3) f32 or NULL, mid_theta / theta (k,) f64.
 * out (k+4) f64 (caller-zeroed): weight_totals[k], sum pm, sum pm * centre (3), with
 * pm_i = w_i . mid_theta and centre_i = p_i - (w_i . theta / 2) n_i (lam b^2 applied by the host). */
int pf_integrate_partials(const double* weights, int64_t n, int32_t k, const float* positions,
                          const float* normals, const double* mid_theta, const double* theta,
                          double* out, void* stream);

/* ---------------------------------------------------------------------------------------------
 * The fused path: project -> depth test -> bilinear gather -> cross-view mean -> L2 normalise ->
 * cosine similarity vs K text embeddings -> temperature softmax -> property regression ->
 * voxel + integrate_mass partials, one pass over the points.
 * ------------------------------------------------------------------------------------------- */

#define PF_FUSE_WRITE_FEATURES 1u  /* validation: write mean features (n,d) f32            */
#define PF_FUSE_WRITE_SIMS 2u      /* validation: write similarities (n,k) f32             */
#define PF_FUSE_WRITE_WEIGHTS 4u   /* validation: write softmax weights (n,k) f32          */
#define PF_FUSE_SKIP_VOXELS 8u     /* do not touch the voxel grid (codes still written)    */
#define PF_FUSE_FORCE_SIMT 16u     /* use the SIMT gather even where the tensor path applies */
#define PF_FUSE_PREPARED 32u       /* workspace already holds pf_fuse_prepare's tables: skip it */
#define PF_FUSE_DETERMINISTIC 128u /* tile path: stable radix sort of the points (run-to-run identical
                                      tiles and results; the default counting sort orders the points of
                                      one sort cell differently per run, a ~1e-6 effect on properties) */
#define PF_FUSE_FEATURE_KERNEL 64u /* bf16 maps: the feature-product tile kernel (k_tile_ws) instead
                                      of the Gram kernel (always taken with PF_FUSE_WRITE_FEATURES) */

/* Number of doubles in the `partials` output of pf_fuse_query. Layout:
 * [0,k)          weight_totals_k = sum_i w_ik                       (integrate.py:133)
 * k              sum_i pm_i,  pm_i = sum_k w_ik * mid_k * theta_k   (integrate.py:146 / (lam b^2))
 * k+1..k+3       sum_i pm_i * x_i                                   (integrate.py:153)
 * k+4            featured point count (visible in >= 1 view)
 * k+5            visible point-view pairs                                                     */
#define PF_PARTIALS_LEN(k) ((k) + 6)

typedef struct pf_fuse_args {
  /* inputs */
  const float* points;      /* (n,3) f32 (bundle.py:158)                                         */
  int64_t n;
  const pf_view_t* views;   /* (nviews) device                                                   */
  const pf_view_t* views_host; /* the same (nviews) records in host memory (launch sizing)       */
  int32_t nviews;
  const float* depth;       /* packed f32 depth maps                                             */
  const void* fmap;         /* packed (Hf,Wf,D) maps, fmap_dtype                                 */
  int32_t fmap_dtype;       /* PF_F32 | PF_BF16                                                  */
  int32_t d;                /* feature dim, d % 8 == 0, d <= 1024 (SIMT)                         */
  const float* text;        /* (k,d) f32 unit rows (grounding.py:86-93)                          */
  int32_t k;                /* materials, k <= 256                                               */
  const float* values;      /* (k,p) f32 property table, column `density_col` is density         */
  int32_t p;                /* properties, p <= 4                                                */
  int32_t density_col;
  const float* mid_theta;   /* (k,) f32 mid_density_k * thickness_k (integrate.py:132,146)       */
  double temperature;       /* softmax T > 0 (grounding.py:168-178)                              */
  double eps;               /* depth tolerance (geometry.py:89-103)                              */
  int32_t grid;             /* voxel grid side g                                                 */
  const double* lo_hi;      /* (6,) voxel domain (pf_bbox), device                               */
  uint32_t flags;           /* PF_FUSE_*                                                         */
  /* outputs */
  int32_t* counts;          /* (n,) visible views per point                                      */
  uint32_t* mask_bits;      /* (n, ceil(nviews/32)) visibility bitset, bit j of word w = view 32w+j */
  float* props;             /* (n,p) regressed properties; zero rows for featureless points      */
  int32_t* codes;           /* (n,) voxel code                                                   */
  float* grid_partials;     /* (2*g^3) f32 [sum rho | count], caller-zeroed unless SKIP_VOXELS   */
  double* partials;         /* (PF_PARTIALS_LEN(k)) caller-zeroed, accumulated                   */
  int32_t* status;          /* (1,) device int32, caller-zeroed; bit0 = NaN similarity seen,     *
                             * bit1 = non-finite softmax sum (inf inputs)                        */
  float* features;          /* optional (n,d) f32 mean features (flag WRITE_FEATURES)            */
  float* sims;              /* optional (n,k) f32 (flag WRITE_SIMS)                              */
  float* weights;           /* optional (n,k) f32 (flag WRITE_WEIGHTS)                           */
  /* scratch */
  void* workspace;          /* pf_fuse_workspace_bytes(args) bytes, 256-byte aligned             */
  /* optional touched-voxel list (2n int32): slots [0,n) per sorted point (voxel code or -1), slots
   * [n, n + *vox_count) appended by the SIMT kernel                                             */
  int32_t* vox_list;        /* (2n,) or NULL                                                     */
  int32_t* vox_count;       /* (1,) device int32, caller-zeroed                                  */
  /* optional staged inputs: cudaEvent_t handles recorded after the upload of the depth maps /
   * of the feature maps and text table (NULL: ready when the call is enqueued). The call then waits
   * for the depth maps only before the visibility stage and for the feature maps only before the G
   * table and the feature gather, so an object's point sort overlaps its own remaining uploads.
   * Points, view records, values and mid_theta must be ready when the call is enqueued.       */
  void* depth_ready;
  void* fmap_ready;
} pf_fuse_args_t;

uint64_t pf_fuse_workspace_bytes(const pf_fuse_args_t* args);
/* Per-object tables into the workspace: G = fmap @ text^T over every feature cell (the similarity
 * by associativity, see csrc/pf_fused.cu). pf_fuse_query runs it itself unless PF_FUSE_PREPARED. */
int pf_fuse_prepare(const pf_fuse_args_t* args, void* stream);
int pf_fuse_query(const pf_fuse_args_t* args, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Capture-bundle ingest, host only: the reference's blob formats into caller-provided
 * (pinned) host buffers; the caller uploads them (paper_2511_03126_b200/ingest.py).
 * ------------------------------------------------------------------------------------------- */

/* TB32 blob header (tensorio.read_tensor, tensorio.py:40-64): rank and dims[4] (0 past the rank).
 * PF_ERR_LOAD if missing, PF_ERR_STRUCTURE with the reference's messages if malformed. */
int pf_tb32_info(const char* path, int32_t* rank, int64_t* dims);
/* TB32 payload (little-endian f32, rank-major) into dst (capacity floats). */
int pf_tb32_read(const char* path, float* dst, int64_t capacity);
/* binary_little_endian PLY (ply.read_ply, ply.py:80-139): vertex count and whether red/green/blue
 * exist. */
int pf_ply_info(const char* path, int64_t* n, int32_t* has_colors);
/* x, y, z -> positions (n, 3) f32; colors (n, 3) u8 when non-null and present. */
int pf_ply_read_points(const char* path, float* positions, uint8_t* colors, int64_t capacity);

/* Workspace bytes of pf_estimate_normals for n points. */
uint64_t pf_normals_workspace_bytes(int64_t n);
/* geometry.estimate_normals (geometry.py:106-146): per point the k nearest points (self included,
 * exact grid search), their mean-centred covariance / k, the unit eigenvector of the smallest
 * eigenvalue oriented so that n . (centroid - p) >= 0 with centroid = (ccx, ccy, ccz) the mean camera
 * centre; neighbourhoods of rank < 2 (lambda_1 <= 1e-10 lambda_2) fall back to the camera direction
 * and are flagged. normals (n, 3) f64, degenerate (n) u8. k in {3, 4, 6, 8, 10, 12, 16, 20, 24, 32},
 * k <= n (PF_ERR_VALUE otherwise, as the reference's ValueError). */
int pf_estimate_normals(const float* points, int64_t n, int32_t k, double ccx, double ccy, double ccz,
                        double* normals, uint8_t* degenerate, void* workspace, void* stream);

/* view_select.score_views + rank_views (view_select.py:51-124) for s anchors x nviews: (s, nviews)
 * s_total / s_angle / z and (s, nviews, 2) pixels, f64; ranked (s, k) i32 = the k best visible
 * views (visibility & z > 0) by (-s_total, view index), -1 padded. visibility (s, nviews) u8. */
int pf_score_views(const double* positions, const double* normals, int64_t s, const pf_view_t* views,
                   int32_t nviews, const uint8_t* visibility, double* s_total, double* s_angle, double* z,
                   double* pixels, int32_t k, int32_t* ranked, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Densification, fp64 like the reference.
 * ------------------------------------------------------------------------------------------- */

/* Workspace bytes of pf_dino_knn_interpolate for nq queries x ns sources (the (nq, ns) similarity
 * matrix dominates). */
uint64_t pf_dino_knn_workspace_bytes(int64_t nq, int64_t ns, int32_t d);
/* densify.dino_knn_interpolate (densify.py:36-86): out (nq, m) = convex combination of the probs
 * rows of each query's k most cosine-similar sources (order: similarity desc, index asc; weights
 * max(sim, 0) renormalised, uniform when all vanish). q (nq, d), s (ns, d), probs (ns, m) f64
 * row-major. neighbors (nq, k) i32 optional. PF_ERR_VALUE if k outside 1..ns; PF_ERR_MATERIAL
 * listing the first zero query rows (densify.py:62-64) — that check synchronises the stream. */
int pf_dino_knn_interpolate(const double* q, int64_t nq, const double* s, int64_t ns, int32_t d,
                            const double* probs, int32_t m, int32_t k, double* out, int32_t* neighbors,
                            void* workspace, void* stream);
/* idx[i] = the point of `points` (np, 3) f64 nearest to queries[i] (fp64 squared distance, lowest
 * index on ties): the cKDTree k=1 donor query of densify_field's featureless points
 * (densify.py:142-147). np == 0 -> PF_ERR_MATERIAL. */
int pf_nearest_index(const double* queries, int64_t nq, const double* points, int64_t np, int64_t* idx,
                     void* stream);
/* The same result through a uniform grid over `points` (exact shell search, O(n) instead of
 * O(nq * np)); workspace pf_nearest_workspace_bytes(np). */
uint64_t pf_nearest_workspace_bytes(int64_t np);
int pf_nearest_index_grid(const double* queries, int64_t nq, const double* points, int64_t np, int64_t* idx,
                          void* workspace, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Cell-range sharding of one object across ranks (SURVEY §8e "shard by voxel-code ranges after a
 * pre-sort"; replaces the dense voxel all-reduce of point-range sharding, pipeline.py:304-312 /
 * integrate.py:133-155 are the per-object reductions it feeds). csrc/pf_shard.cu describes the
 * protocol; the collectives between the calls belong to the caller (dist.py: NCCL or in-process).
 * ------------------------------------------------------------------------------------------- */

/* Number of histogram bins (64^3 cells) used by pf_shard_keys / pf_shard_cuts. */
int32_t pf_shard_bins(void);
/* keys[i] = Hilbert index of the 64^3 cell enclosing point i's voxel (voxel code of the fused path,
 * cell_a = code_a * 64 / g); hist[key] += 1 (hist: pf_shard_bins() u32, zeroed by the caller). */
int pf_shard_keys(const float* points, int64_t n, const double* lo_hi, int32_t g, uint32_t* keys, uint32_t* hist,
                  void* stream);
/* cuts (world + 1) u32: rank r owns cells [cuts[r], cuts[r+1]) — balanced split of the GLOBAL
 * (all-reduced) histogram along the curve. world in [1, 64]. */
int pf_shard_cuts(const uint32_t* hist, int32_t world, uint32_t* cuts, void* stream);
/* Group the local points by owner: counts (world) i32, cursor (world) i32 scratch, send (n) float4
 * {x, y, z, local index bits}, destination blocks contiguous in rank order. */
int pf_shard_pack(const float* points, int64_t n, const uint32_t* keys, const uint32_t* cuts, int32_t world,
                  int32_t* counts, int32_t* cursor, void* send, void* stream);
/* Received float4 points -> (n, 3) f32. */
int pf_shard_xyz(const void* recv, int64_t n, float* xyz, void* stream);
/* Per-point results -> int32 rows [props (p, f32 bits) | count | code | mask (nwords)]. */
int pf_shard_pack_results(int64_t n, int32_t p, int32_t nwords, const float* props, const int32_t* counts,
                          const int32_t* codes, const int32_t* mask, int32_t* rows, void* stream);
/* Returned rows (in the order the points were sent) -> caller-order outputs, by the local index each
 * sent float4 carried. */
int pf_shard_unpack_results(int64_t n, int32_t p, int32_t nwords, const int32_t* rows, const void* sent,
                            float* props, int32_t* counts, int32_t* codes, int32_t* mask, void* stream);

/* Fixed-capacity exchange (no host synchronisation; graph-capturable with NCCL collectives): the
 * send buffer is world blocks of (capacity + 1) float4, row 0 of block o = {count (int bits),
 * flags (int bits), 0, 0} and rows 1.. the points for owner o ({x, y, z, local index bits});
 * unused rows are NaN points, which the fused path treats as padding slots (invisible, voxel code
 * -1, no voxel or partial contribution). An owner receiving more than `capacity` points from this
 * rank sets flags bit 0 (the surplus is dropped: the caller re-runs with a larger capacity or the
 * count-exchanging pf_shard_pack). cursor: world i32 scratch; flags: one device i32. After an
 * equal-split all-to-all of the blocks: */
int pf_shard_pack_padded(const float* points, int64_t n, const uint32_t* keys, const uint32_t* cuts, int32_t world,
                         int32_t capacity, int32_t* cursor, void* send, int32_t* flags, void* stream);
/* received blocks -> (world * capacity, 3) f32 in slot order (padding rows NaN), the input of a
 * fixed-size pf_fuse_query; */
int pf_shard_unpad(const void* recv, int32_t world, int32_t capacity, float* xyz, void* stream);
/* and, after the reverse equal-split all-to-all of pf_shard_pack_results rows (world * capacity
 * rows, slot order), the rows of the points this rank sent (row 0 counts of `sent`) -> caller order. */
int pf_shard_unpack_results_padded(int32_t world, int32_t capacity, int32_t p, int32_t nwords, const int32_t* rows,
                                   const void* sent, float* props, int32_t* counts, int32_t* codes, int32_t* mask,
                                   void* stream);

/* The per-object reductions over NCCL for C/C++ hosts (integrate.py:133-155 partials +
 * the voxel grid of point-range sharding): in-place sum of grid_partials (n_grid f32, may be 0) and
 * partials (n_partials f64) over `comm` (an ncclComm_t) on `stream`. NCCL is resolved at run time
 * (dlopen libnccl.so.2, preferring the copy already loaded in the process). */
int pf_allreduce_partials(float* grid_partials, int64_t n_grid, double* partials, int64_t n_partials, void* comm,
                          void* stream);
/* A one-rank NCCL communicator (loopback tests of pf_allreduce_partials); destroy with the call below. */
int pf_nccl_comm_init_single(void** comm);
int pf_nccl_comm_destroy(void* comm);

/* ---------------------------------------------------------------------------------------------
 * Diagnostics (no reference twin).
 * ------------------------------------------------------------------------------------------- */

/* Stage timer of the tensor-core tile path: enable (1) / disable (0) CUDA-event marks at the stage
 * boundaries of every following pf_fuse_query (resets the record). pf_stage_times then fills
 * ms[0..4] with the summed device time of sort, prep, tile kernel, unsort and SIMT overflow over
 * the recorded calls (synchronising on their events) and returns the number of calls (<= 64), or
 * minus a PF_ERR_* status. */
int pf_stage_timing(int32_t enable);
/* tcgen05.mma rate microbenchmark: per SM, reps x 8 MMAs (M=128, N=n, K=16, A from shared memory or
 * TMEM (ts), B resident in shared memory), optionally with concurrent shared-memory stores; writes
 * (issue cycles, issue->completion cycles) per SM to out_dev (2 x SMs uint64). */
int pf_bench_umma(int32_t n, int32_t ts, int32_t reps, int32_t stores, void* out_dev, void* stream);
/* B-operand loader microbenchmark: per SM, `stages` x 16 KB of 128-byte rows gathered from a
 * (cells, 1024) bf16 table with cp.async (mode 0, the tile kernel's loader pattern) or TMA
 * tile::gather4 (mode 1); writes cycles per SM to out_dev (SMs uint64). */
int pf_bench_gather(const void* src_bf16, int32_t cells, int32_t stages, int32_t mode, void* out_dev, void* stream);
int pf_stage_times(float* ms, int32_t n);
/* tcgen05 FLOPs the last pf_fuse_query on args' workspace issued in the tile kernel (ktp = a work
 * item's taps padded to 16): feature-product kernel 2 * 128 * ktp * (D + 128) per item; Gram kernel
 * 2 * 128 * ktp * D (+ the taps-128.. block) per item + 2 * 128 * ktp * (128 + ktp) per 128-row
 * block; 0 for the SIMT path. Synchronises the stream. */
int pf_tile_executed_flops(const pf_fuse_args_t* args, double* flops, void* stream);
/* The tile path's point-sort key: the 24-state automaton of the 3-D Hilbert curve (Skilling's
 * transpose algorithm), entry [state * 8 + octant] = key digit | 8 * next state, root state 0.
 * pf_hilbert_table copies its 192 bytes to host memory `out` (n >= 192) and returns the state count;
 * pf_hilbert_keys writes the key of every point's cell of the 2^bits grid (bits 7 or 8) over the
 * bbox lo_hi (the sort's cell mapping) to keys (n,) uint32 on the device. */
int pf_hilbert_table(uint8_t* out, int32_t n);
int pf_hilbert_keys(const float* points, int64_t n, const double* lo_hi, int32_t bits, uint32_t* keys,
                    void* stream);

/* C (128,n) f32 = A (128,k) bf16 row-major @ B (k,n) bf16 row-major through the tile kernel's
 * tcgen05 operand layouts / descriptors / TMEM read-back. k % 64 == 0 (<= 256), n % 16 == 0.
 * ts != 0: A is first copied to TMEM with tcgen05.cp and the MMAs read A from TMEM. */
int pf_selftest_umma(const void* a_bf16, const void* b_bf16, float* c, int32_t k, int32_t n,
                     int32_t ts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PROPFIELD_B200_H */

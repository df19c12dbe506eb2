/*
 * glod_b200 — C ABI of the B200-native per-view hot path of
 * "A LoD of Gaussians" (arXiv 2507.01110).
 *
 * Plain C: pointers, sizes and a cudaStream_t passed as void*.  Every
 * pointer marked [dev] is device memory owned by the caller; the library
 * owns nothing between calls (scratch is caller-provided, sized by the
 * matching *_scratch_bytes query).  All work is enqueued on `stream`;
 * nothing synchronises unless stated.  Every call returns GLOD_OK (0) or an
 * error code; glod_last_error() returns a thread-local message.
 *
 * The reference (/root/reference/pkg/src/glod, pure Python) has no FFI: its
 * boundary is its Python function signatures.  Each entry point below cites
 * the reference function it replaces; the Python mirror in
 * paper_2507_01110_b200/ binds these through ctypes.
 */
#ifndef GLOD_B200_H
#define GLOD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference exception classes) ---------- */
#define GLOD_OK 0
#define GLOD_ERR_INVALID_ARGUMENT 1   /* ValueError / InvalidParameterError */
#define GLOD_ERR_CUDA 2               /* RuntimeError                        */
#define GLOD_ERR_INVALID_INPUT 3      /* renderer.InvalidInputError          */
#define GLOD_ERR_OVER_BUDGET 4        /* cache.OverBudgetError               */

int glod_version(void);
const char* glod_last_error(void);
/* Number of kernels this library has launched in the process so far. */
uint64_t glod_launch_count(void);

/* ======================================================================= *
 * LoD selection
 * ======================================================================= */

/* Static per-HSPT scene data (uploaded once per HSPT version). */
typedef struct glod_lod_scene {
  int64_t capacity;             /* hierarchy node slots                       */
  int32_t root;                 /* Hierarchy.root                             */
  int32_t attr_stride;          /* doubles between consecutive nodes' means /
                                   scales: 0 or 3 = dense [capacity*3];
                                   GLOD_NODE_RECORD = node records          */
  const int32_t* children;      /* [dev] [capacity*2], -1 = NONE              */
  const int32_t* kind;          /* [dev] [capacity]: spt_id>=0 | -2 pass | -1 */
  const double* means;          /* [dev] live f64 means (see attr_stride)     */
  const double* scales;         /* [dev] live f64 scales                      */
  int32_t num_spts;
  int32_t key_f64;              /* 1: f64 keys, 0: f32 keys (file scenes)     */
  int64_t num_records;          /* total SPT records                          */
  const int64_t* spt_offset;    /* [dev] [S] first record of each SPT         */
  const int32_t* spt_count;     /* [dev] [S]                                  */
  const int32_t* spt_root_rec;  /* [dev] [S] record index of the SPT root     */
  const double* spt_center;     /* [dev] [S*3] Spt.root_center (build time)   */
  const void* key_self;         /* [dev] [R] f32|f64                          */
  const void* key_parent;       /* [dev] [R] f32|f64, descending per SPT      */
  const int32_t* rec_node;      /* [dev] [R] node id of each record           */
  /* optional (NULL / 0: level-synchronous BFS): the candidate nodes a cut
   * can visit — every node reachable from root without entering an SPT
   * subtree (upper nodes, SPT roots, passthrough subtrees) — and the parent
   * array.  With them the select evaluates every candidate at once (its own
   * cull / take test, then a walk up its ancestor chain) instead of one
   * grid barrier per BFS level. */
  const int32_t* parent;        /* [dev] [capacity], -1 = NONE                */
  const int32_t* cand;          /* [dev] [num_cand]: first the upper-BFS nodes
                                   (upper nodes, SPT roots, passthrough roots),
                                   then the passthrough-subtree members     */
  int64_t num_cand;
  int64_t num_cand_upper;
} glod_lod_scene;

/* Per-view parameters: camera position, frustum planes computed on the host
 * with Frustum.from_camera (core.py:301-328), LodConfig. */
typedef struct glod_lod_view {
  double position[3];
  double planes[24];            /* 6 x (nx, ny, nz, d)                        */
  int32_t cull;
  int32_t metric;               /* 0 max_scale, 1 surface_area                */
  double threshold;
} glod_lod_view;

typedef struct glod_lod_select_out {
  int32_t* upper_ids;           /* [dev] [capacity] sorted                    */
  int32_t* pass_ids;            /* [dev] [capacity] sorted                    */
  int32_t* spt_ids;             /* [dev] [S] sorted selected spt ids          */
  double* d_root;               /* [dev] [S]                                  */
  int32_t* prefix_len;          /* [dev] [S]                                  */
  int32_t* counts;              /* [dev] [4] n_upper, n_pass, n_spt, levels   */
} glod_lod_select_out;

/* Replaces hspt.cut_hspt stage 1 + stage-2 prologue (hspt.py:104-153) and
 * the passthrough hierarchy.bfs_cut calls (hierarchy.py:244-266). */
int64_t glod_lod_select_scratch_bytes(int64_t capacity, int32_t num_spts);
int glod_lod_select(const glod_lod_scene* scene, const glod_lod_view* view,
                    const glod_lod_select_out* out, void* scratch,
                    int64_t scratch_bytes, void* stream);

typedef struct glod_spt_compact_in {
  const int32_t* n_spt;         /* [dev] scalar                               */
  const int32_t* spt_ids;       /* [dev] [n_spt]                              */
  const double* dist;           /* [dev] [n_spt] cut distance per SPT         */
  const int32_t* known_prefix;  /* [dev] [n_spt] #{key_parent > dist} when the
                                   caller already has it (select output, cache
                                   entry), or NULL: binary search            */
} glod_spt_compact_in;

typedef struct glod_spt_compact_out {
  int32_t* prefix_len;          /* [dev] [S]                                  */
  int32_t* root_rule;           /* [dev] [S]                                  */
  int64_t* seg_start;           /* [dev] [S]                                  */
  int32_t* sel_seg;             /* [dev] [R] segment (index into spt_ids)     */
  int32_t* sel_pos;             /* [dev] [R] record position within the SPT   */
  int32_t* sel_node;            /* [dev] [R] node id                          */
  int64_t* total;               /* [dev] [2] n_selected, virtual length       */
} glod_spt_compact_out;

/* Replaces spt.cut_spt (spt.py:67-75) for a batch of SPTs and
 * trainer._spt_positions (trainer.py:302-309). */
int64_t glod_spt_compact_scratch_bytes(int32_t num_spts, int64_t num_records);
int glod_spt_compact(const glod_lod_scene* scene, const glod_spt_compact_in* in,
                     const glod_spt_compact_out* out, void* scratch,
                     int64_t scratch_bytes, void* stream);

/* ---- HSPT / SPT build -------------------------------- */
typedef struct glod_hspt_build_in {
  int64_t capacity;             /* hierarchy node slots                       */
  int32_t root;                 /* Hierarchy.root                             */
  int32_t min_subtree;          /* build_hspt min_subtree (>= 1)              */
  const int32_t* parent;        /* [dev] [capacity], -1 = NONE                */
  const int32_t* children;      /* [dev] [capacity*2], -1 = NONE              */
  const double* means;          /* [dev] [capacity*3]                         */
  const double* scales;         /* [dev] [capacity*3]                         */
  double size_threshold;        /* volume threshold (> 0)                     */
  double lod_threshold;         /* LodConfig.threshold used for the keys      */
  int32_t metric;               /* 0 max_scale, 1 surface_area                */
  int32_t corrected;            /* build_spt(corrected=...)                   */
} glod_hspt_build_in;

typedef struct glod_hspt_build_out {
  int32_t* upper_ids;           /* [dev] [capacity] ascending                 */
  int32_t* pass_ids;            /* [dev] [capacity] ascending passthrough roots */
  int32_t* spt_roots;           /* [dev] [capacity] ascending = spt_id order  */
  int32_t* spt_count;           /* [dev] [capacity] records per SPT           */
  int64_t* spt_offset;          /* [dev] [capacity] first record of each SPT  */
  int32_t* rec_node;            /* [dev] [capacity] record node ids           */
  double* key_self;             /* [dev] [capacity]                           */
  double* key_parent;           /* [dev] [capacity] (+inf at each SPT root)   */
} glod_hspt_build_out;

/* Replaces hspt.build_hspt (hspt.py:64-93) with spt.build_spt (spt.py:45-64)
 * for every SPT root, bit-exact (same lists, record order and f64 keys).
 * Synchronises the stream once; sizes[4] (host) = {n_upper, n_pass, n_spt,
 * n_records}.  Free / unreachable node slots belong to no list. */
int64_t glod_hspt_build_scratch_bytes(int64_t capacity);
int glod_hspt_build(const glod_hspt_build_in* in, const glod_hspt_build_out* out, void* scratch,
                    int64_t scratch_bytes, int64_t* sizes, void* stream);

/* ======================================================================= *
 * Rasteriser (renderer.py)
 * ======================================================================= */

/* Pinhole camera, resolved on the host: w2c = Camera.world_to_cam
 * (quat_to_rotmat(orientation).T, core.py:285-287), row-major. */
typedef struct glod_camera {
  double position[3];
  double w2c[9];
  double fx, fy, cx, cy;
  double near_plane;
  int32_t width, height;
} glod_camera;

/* Opaque per-device rasteriser context: owns its stream-ordered workspace
 * and the forward state the backward pass consumes. */
typedef struct glod_raster glod_raster;

typedef struct glod_render_stats {
  int64_t n_gaussians;          /* rows in the render set                    */
  int64_t n_instances;          /* (gaussian, 16x16 tile) pairs              */
  int32_t tiles_x, tiles_y;
  int32_t depth_full_sort;      /* 1: near-tied depths formed long runs and the
                                   depth order was finished with full-width
                                   radix passes (K6)                          */
  int32_t reserved;
} glod_render_stats;

int glod_raster_create(glod_raster** out);
int glod_raster_destroy(glod_raster* r);

/* Replaces render_forward (renderer.py:117-166).  attrs: [dev] packed f64
 * attribute block of n rows, section-major [means 3n | scales 3n |
 * rotations 4n | opacities n | base_colors 3n | sh_rest 9n].  image: [dev]
 * f32 (height, width, 3).  Synchronises once (instance count, finiteness
 * check: GLOD_ERR_INVALID_INPUT names the first non-finite Gaussian like
 * renderer._check_finite). */
int glod_render_forward(glod_raster* r, const double* attrs, int64_t n,
                        const glod_camera* cam, float* image, void* stream);

/* Frame pipelining (no reference counterpart; same images): with deferral
 * enabled, glod_render_forward(_plan) enqueues everything up to the
 * compositing kernel and returns; glod_render_blend enqueues the blend of
 * that forward (GLOD_ERR_INVALID_ARGUMENT if none is pending).  A caller
 * puts independent work — the next frame's LoD select — between the two so
 * its host read-back is not queued behind the blend.  glod_render_backward
 * fails while a blend is pending. */
int glod_render_defer_blend(glod_raster* r, int32_t enable);
int glod_render_blend(glod_raster* r, void* stream);

/* Replaces backward (renderer.py:197-304) for the last forward call.
 * dl_dimage: [dev] f32 (height, width, 3).  grads: [dev] packed f64 block
 * of n rows (same layout as attrs; raw scale/opacity, not log/logit). */
int glod_render_backward(glod_raster* r, const float* dl_dimage, double* grads, void* stream);

int glod_render_stats_get(const glod_raster* r, glod_render_stats* out);
/* Optional CUDA-event timing of the blend kernels (measurement only; no
 * reference counterpart).  Collects finished launches into
 * ms_out[2] = {Σ forward blend ms, Σ backward blend ms} and
 * launches_out[2]; then enable >= 0 resets the sums and turns timing on
 * (1) or off (0); enable < 0 leaves both as they are. */
int glod_render_blend_timing(glod_raster* r, int32_t enable, double* ms_out, int64_t* launches_out);
/* The same with the preprocess kernel (K5, or K4+K5 fused) as a third
 * entry: ms_out[3], launches_out[3]. */
int glod_render_kernel_timing(glod_raster* r, int32_t enable, double* ms_out, int64_t* launches_out);

/* Replaces loss (renderer.py:322-360): (1-lam)*L1 + lam*(1-SSIM), 11-tap
 * sigma=1.5 window, zero padding.  rendered/target/grad: [dev] f32
 * (height, width, 3).  value: [dev] f64[3] = {loss, l1, mean ssim}. */
int64_t glod_loss_scratch_bytes(int32_t width, int32_t height);
int glod_loss_l1_ssim(const float* rendered, const float* target, int32_t width,
                      int32_t height, double lam, double* value, float* grad,
                      void* scratch, int64_t scratch_bytes, void* stream);

/* ======================================================================= *
 * Optimiser (trainer._adam_update, trainer.py:253-299)
 * ======================================================================= */

/* Node records: the training engine's master layout, one 576-B (18-sector)
 * record per node, f64 [capacity][GLOD_NODE_RECORD]:
 *   [0, 23)   attribute values (means 3 | scales 3 | rotations 4 | opacity |
 *             base_colors 3 | sh_rest 9)
 *   [24, 70)  ADAM moments, (m, v) per attribute value (16-B aligned pairs)
 *   70        per-node step count (int64 bits)
 *   23, 71    padding
 * so one ADAM update reads and writes whole records, and the LoD kernels read
 * means/scales at stride GLOD_NODE_RECORD (glod_lod_scene.attr_stride). */
#define GLOD_NODE_RECORD 72
#define GLOD_REC_MV 24
#define GLOD_REC_STEP 70

/* One ADAM step, in place, on params[ids] from grads[rows]
 * (trainer._adam_update, trainer.py:253-299).  params: [dev] packed f64
 * block of `capacity` rows (section-major, as h.attrs).  mv: [dev] the ADAM
 * moments (OptimizerState m/v, trainer.py:93-124) row-major and
 * interleaved: f64 [capacity][23][2] = {m, v} per attribute value, so one
 * node's moments are 368 contiguous bytes.  step: [dev] int64[capacity];
 * grads: [dev] packed f64 block of `grad_rows` rows; ids/rows: [dev]
 * int32[n] (rows == NULL means row i).  ids must be unique.  lrs: host
 * double[6] in section order (means already scaled by the scene extent).
 * bias_table: [dev] f64 [2*bias_len] = {1-0.9^t, 1-0.999^t for t <
 * bias_len} (or NULL / bias_len 0: computed with pow in the kernel).
 * refresh (optional, see glod_gather_plan below): when given, row r is a
 * render row of that plan and SPT rows also write their updated values
 * into their cache block (entry.block.attrs.put, trainer.py:363). */
struct glod_gather_plan;
int glod_adam_step(double* params, double* mv, int64_t* step, int64_t capacity,
                   const int32_t* ids, const double* grads, const int32_t* rows,
                   int64_t grad_rows, int64_t n, const double* lrs, const double* bias_table,
                   int64_t bias_len, const struct glod_gather_plan* refresh, void* stream);
/* The same step on node records (GLOD_NODE_RECORD layout above): params,
 * moments and step count of a node are one contiguous record; the step
 * counts are incremented in the same launch. */
int glod_adam_step_records(double* records, int64_t capacity, const int32_t* ids, const double* grads,
                           const int32_t* rows, int64_t grad_rows, int64_t n, const double* lrs,
                           const double* bias_table, int64_t bias_len,
                           const struct glod_gather_plan* refresh, void* stream);

/* ======================================================================= *
 * Store / cache data movement (trainer.py:325-364, store.py:304-333)
 * ======================================================================= */

/* Where each render row comes from: rows [0, n_upper+n_pass) are master
 * rows (h.attrs.take(concat(upper, passthrough))); row n_upper+n_pass+k is
 * row sel_pos[k] of the cache block of segment sel_seg[k].  Blocks and the
 * master are packed f64 attribute blocks (seg_rows[j] / capacity rows). */
typedef struct glod_gather_plan {
  double* master;               /* [dev] packed f64, capacity rows            */
  int64_t capacity;
  const int32_t* upper_ids;     /* [dev] [n_upper]                            */
  const int32_t* pass_ids;      /* [dev] [n_pass]                             */
  int32_t n_upper;
  int32_t n_pass;
  const int32_t* sel_seg;       /* [dev] [n_sel] (glod_spt_compact output)    */
  const int32_t* sel_pos;       /* [dev] [n_sel]                              */
  const int32_t* sel_node;      /* [dev] [n_sel]                              */
  int64_t n_sel;
  const uint64_t* seg_block;    /* [dev] [n_spt] device address of each block */
  const int64_t* seg_rows;      /* [dev] [n_spt] rows (prefix_len) per block  */
  int64_t master_stride;        /* 0: master is a packed section-major block;
                                   GLOD_NODE_RECORD: node records            */
  int32_t spt_from_master;      /* 1: SPT rows read from the master too (view-
                                   sharded training: the replicated node
                                   records are authoritative, csrc/exchange.cu) */
} glod_gather_plan;

/* AttributeArrays.concat of the render set into `out` (packed f64, R =
 * n_upper+n_pass+n_sel rows); row_node (optional) receives each row's node. */
int glod_gather_render_rows(const glod_gather_plan* plan, double* out, int32_t* row_node,
                            void* stream);
/* glod_gather_render_rows fused into glod_render_forward: the rasteriser
 * reads render row r from the source the gather would copy it from (so the
 * image, the finiteness check and the following glod_render_backward are
 * those of glod_render_forward on the gathered rows) and writes row_node[r];
 * the packed render-set copy is never made.  R = n_upper+n_pass+n_sel.  The
 * plan's device arrays, blocks and master must stay unchanged until the
 * matching glod_render_backward has run. */
int glod_render_forward_plan(glod_raster* r, const glod_gather_plan* plan, int32_t* row_node,
                             const glod_camera* cam, float* image, void* stream);
/* entry.block.attrs.put(pos, h.attrs.take(node_ids)) for every SPT row. */
int glod_scatter_to_blocks(const glod_gather_plan* plan, void* stream);
/* Serve path: wire payloads of the cut-delta protocol
 * (protocol._wire_attrs, protocol.py:40-49; encode_spt_load /
 * encode_upper_set :80-92).  Message k covers ids[seg_start[k] ..
 * seg_start[k+1]) and is written at out + 23*seg_start[k] as the
 * section-major little-endian f32 SoA [means 3n | scales 3n | rotations 4n
 * | opacities n | base_colors 3n | sh_rest 9n] of master rows (f64 ->
 * f32 round-to-nearest, as astype("<f4")).  master: [dev] packed f64,
 * capacity rows; ids: [dev] int32 [n_rows]; seg_start: [dev] int64
 * [n_msgs+1]; out: [dev] or mapped pinned host (glod_host_device_ptr),
 * 23*n_rows floats. */
int glod_wire_pack(const double* master, int64_t capacity, const int32_t* ids, const int64_t* seg_start,
                   int32_t n_msgs, int64_t n_rows, float* out, void* stream);
/* View-sharded training (no single-view counterpart): after the replicated
 * ADAM on the union `ids` of every rank's touched nodes, copy each updated
 * master row into this rank's resident cache block holding it — the rule of
 * trainer.py:363 applied to the union.  spt_of_node/rec_of_node: [dev]
 * int32[capacity] (SPT id / record position of each node, -1 if none);
 * res_block/res_rows: [dev] per SPT id, the resident block and its rows
 * (0 if not resident; glod_cache_resident); touched: [dev] int32 per SPT id,
 * set to 1 for every block written (feed to glod_cache_mark_dirty). */
int glod_refresh_resident_blocks(const double* master, int64_t capacity, int64_t master_stride,
                                 const int32_t* ids, int64_t n,
                                 const int32_t* spt_of_node, const int32_t* rec_of_node,
                                 const uint64_t* res_block, const int64_t* res_rows, int32_t* touched,
                                 void* stream);
/* ======================================================================= *
 * K11-exchange: sparse gradient exchange of view-sharded training (SURVEY
 * §8e, csrc/exchange.cu).  No reference counterpart (the reference has no
 * multi-device path); it replaces the python all-reduce of
 * round 1 (parallel.sparse_grad_allreduce).  Contract: the gradient ADAM
 * applies to node i = Σ over ranks of that step's per-view gradients.
 * Ownership: owner(id) = (id >> 5) mod nranks.  U = the union of every
 * rank's render-row ids, laid out owner-major (owner chunks, each sorted).
 * ======================================================================= */
typedef struct glod_xchg glod_xchg;
/* ncclGetUniqueId into 128 bytes (rank 0 creates, the caller broadcasts). */
int glod_nccl_unique_id(void* out128);
/* Exchange context for `nranks` ranks over node ids [0, capacity).  With a
 * unique id, the context owns an NCCL communicator (ncclCommInitRank) and
 * the composed calls below are available; with NULL only the phase calls
 * (transport supplied by the caller). */
int glod_xchg_create(int32_t nranks, int32_t rank, int64_t capacity, const void* nccl_id128,
                     glod_xchg** out);
int glod_xchg_destroy(glod_xchg* x);
/* Phases 1-4 over NCCL: all-gather of the row ids, on-device union,
 * gradients (packed section-major, R rows) bucketed by owner and sent
 * point to point (grouped ncclSend/ncclRecv), summed by the owner source by
 * source.  *n_owned = rows of this rank's chunk (glod_xchg_owned). */
int glod_grad_exchange(glod_xchg* x, const int32_t* row_node, const double* grads, int64_t R,
                       int64_t* n_owned, void* stream);
/* Phase 5 over NCCL: each owner's updated attribute rows (first 23 values
 * of its node records, after ADAM) broadcast; every rank writes all of U
 * into its node records (stride in doubles). */
int glod_param_allgather(glod_xchg* x, double* records, int64_t stride, void* stream);
/* The phases, for a caller-supplied transport.  union: ids_all [dev] n
 * gathered ids (-1 = padding) -> owner_off [host] nranks+1 offsets (syncs). */
int glod_xchg_union(glod_xchg* x, const int32_t* ids_all, int64_t n, int64_t* owner_off, void* stream);
int glod_xchg_union_ids(glod_xchg* x, const int32_t** ids, int64_t* n);
/* pack: this rank's rows bucketed by owner into wire rows of 24 f64
 * (owner-local position, 23 gradients); counts [host] nranks (syncs). */
int glod_xchg_pack(glod_xchg* x, const int32_t* row_node, const double* grads, int64_t R, int64_t* counts,
                   const double** send, void* stream);
int glod_xchg_begin_accumulate(glod_xchg* x, double** acc, int64_t* n_owned, void* stream);
/* add one source's received wire rows (call once per source, rank order) */
int glod_xchg_accumulate(glod_xchg* x, const double* rows, int64_t m, void* stream);
int glod_xchg_owned(glod_xchg* x, const int32_t** ids, const double** grads, int64_t* n);
/* pack_params: this rank's chunk of the |U| x 23 row-major buffer from the
 * node records; scatter_params: all of it back into the node records. */
int glod_xchg_pack_params(glod_xchg* x, const double* records, int64_t stride, double** params, void* stream);
int glod_xchg_scatter_params(glod_xchg* x, double* records, int64_t stride, void* stream);
/* {|U|, owned rows, bytes sent, bytes received} of the last step. */
int glod_xchg_stats(glod_xchg* x, int64_t* out4);

/* Elementwise f32 -> f64 (to_f64=1) or f64 -> f32 (store write-back). */
int glod_convert(const void* in, void* out, int64_t n, int32_t to_f64, void* stream);

/* The pinned host store (store.py's slot-ordered f32 sections), as device-
 * accessible addresses of page-locked host memory (glod_host_device_ptr). */
typedef struct glod_store_view {
  const float* section[6];      /* [host-mapped] first value of section k     */
  int64_t nslots;
  /* 0: section-major (section k is nslots x cols_k, the .glod file's
   * layout); 23: interleaved rows — one 92-B row per slot, section[k] =
   * row base + column offset of k — so an SPT prefix is ONE contiguous
   * range (one copy-engine transfer).  Other values are rejected. */
  int64_t row_stride;
} glod_store_view;

/* One SPT prefix transfer: `rows` slots starting at `slot_start` <-> the
 * packed f64 cache block `block`.  elem_start = 23 * (rows of all earlier
 * items): the items of one call tile a flat index space of 23*sum(rows). */
typedef struct glod_prefix_item {
  int64_t slot_start;
  int64_t rows;
  int64_t elem_start;
  double* block;                /* [dev]                                       */
  /* loads only: rows [0, min(rows, overlay_rows)) are taken as
   * f64(f32(overlay row)) from this packed f64 block of overlay_rows rows
   * instead of the store —
   * a block evicted earlier in the same step whose write-back is in flight
   * (store.py:323-333 then :314-321).  NULL / 0 for a plain load. */
  const double* overlay;        /* [dev]                                       */
  int64_t overlay_rows;
  /* loads only: when non-NULL the prefix is read from this packed f32
   * copy in HBM, laid out like the store (row order for an interleaved
   * store, else section-major; a prefetch, glod_cache_prefetch) instead of
   * the store. */
  const float* src;             /* [dev]                                       */
} glod_prefix_item;

/* Device address of page-locked host memory (cudaHostGetDevicePointer). */
int glod_host_device_ptr(void* host, void** dev);
/* Scene.load_spt_prefix + astype(f64) for a batch of misses (store.py:314-321,
 * trainer.py:333-334): one zero-copy kernel, f32 -> f64.  items: [dev]. */
int glod_store_load_prefixes(const glod_store_view* store, const glod_prefix_item* items,
                             int32_t n_items, int64_t total_elems, void* stream);
/* Scene.write_back for a batch of evicted/flushed blocks (store.py:323-333):
 * f64 -> f32 written straight into the pinned store. */
int glod_store_write_back(const glod_store_view* store, const glod_prefix_item* items,
                          int32_t n_items, int64_t total_elems, void* stream);

/* ======================================================================= *
 * Device cache table (cache.DeviceCache, cache.py:42-109, driven like the
 * gather loop of trainer.train_step, trainer.py:329-345)
 * ======================================================================= */
typedef struct glod_cache glod_cache;

typedef struct glod_cache_stats_t {
  int64_t entries, resident_bytes, hits, misses, loaded_rows;
  int64_t prefetched_rows, prefetch_used_rows;
  int64_t pool_allocs, grow_events;   /* block-arena misses, staging re-allocations */
  int64_t host_ns_step, host_ns_prefetch;  /* host time spent in cache_step / cache_prefetch */
  int64_t pf_copies;                       /* prefetch prefixes issued (one copy each) */
} glod_cache_stats_t;

/* slot_start: host int64[num_spts], first store slot of each SPT
 * (Scene.spt_slot_start, store.py:299-302).  bytes_per_row = 92. */
int glod_cache_create(int64_t budget_bytes, double d_min, double d_max, int64_t flush_interval,
                      int32_t bytes_per_row, const int64_t* slot_start, int32_t num_spts,
                      glod_cache** out);
int glod_cache_destroy(glod_cache* c);
/* One view's cache pass over the selected SPTs (host arrays, ascending
 * spt order): lookup, miss → stream-ordered block allocation + prefix load
 * from the pinned store, insert with LRU eviction and write-back of dirty
 * victims.  Outputs per SPT the distance its positions are cut at
 * (cached_distance), its block address and rows.  counters_out[2] =
 * {rows loaded from the store, cache hits}.  GLOD_ERR_OVER_BUDGET when one
 * prefix exceeds the budget. */
int glod_cache_step(glod_cache* c, const glod_store_view* store, int32_t n,
                    const int32_t* spt_ids, const double* d_root, const int32_t* prefix_len,
                    double* dist_out, uint64_t* block_out, int64_t* rows_out,
                    int64_t* counters_out, void* stream);
/* After the step's kernels are enqueued: mark this step's entries dirty
 * (training), tick_and_maybe_flush(iteration) (iteration < 0: no flush),
 * release evicted blocks stream-ordered. */
int glod_cache_end_step(glod_cache* c, const glod_store_view* store, int64_t iteration,
                        int32_t mark_dirty, void* stream);
/* Prefetch for a predicted view (no reference counterpart: the reference
 * reads the store synchronously inside train_step, trainer.py:333-334).
 * Host arrays as for glod_cache_step.  Every SPT the table would miss
 * right now (lookup semantics of cache.py:56-73, no LRU update) is copied
 * store → f32 HBM buffer by the copy engines on a prefetch stream, after
 * all write-backs issued so far; at most max_rows rows (< 0: no cap).
 * The next glod_cache_step uses a prefetch for a miss with the same prefix
 * length whose store rows were not written back since; the others are
 * freed.  Counters and cache decisions are unaffected.  rows_out: rows
 * issued. */
int glod_cache_prefetch(glod_cache* c, const glod_store_view* store, int32_t n,
                        const int32_t* spt_ids, const double* d_root, const int32_t* prefix_len,
                        int64_t max_rows, int64_t* rows_out, void* stream);
int glod_cache_stats(const glod_cache* c, glod_cache_stats_t* out);
/* Diagnostics: cumulative host ns per glod_cache_step phase (decisions,
 * disk reads, materialize, loads, write-back staging, -, -, -). */
int glod_cache_debug_profile(const glod_cache* c, int64_t* ns_out8);
/* Implicit block refresh.  A cache block holds its prefix's 23*rows f64
 * values (section-major) followed by one "touched" bit per row
 * (ceil(rows/64) u64).  ADAM (glod_adam_step_records with a refresh plan)
 * and glod_refresh_resident_blocks set a row's bit instead of writing the
 * updated master row into the block (entry.block.attrs.put, trainer.py:363):
 * a touched row's value is the master row, and the gather reads it from
 * there.  Before a block is written back to the store (or overlaid by a
 * reload) its touched rows are materialised from the master, which this
 * call registers: master rows (packed section-major when master_stride = 0,
 * else node records of that stride), the record node ids (rec_node, [dev],
 * the LoD scene's) and each SPT id's first record (host int64[num_spts]). */
int glod_cache_set_master(glod_cache* c, const double* master, int64_t capacity, int64_t master_stride,
                          const int32_t* rec_node, const int64_t* rec_offset, int32_t num_spts);
/* Materialise every resident block now (snapshots / tests). */
int glod_cache_materialize(glod_cache* c, void* stream);
/* Host tables of the resident blocks per SPT id (block address, rows; 0 if
 * not resident), for glod_refresh_resident_blocks. */
int glod_cache_resident(const glod_cache* c, uint64_t* block, int64_t* rows, int32_t num_spts);
/* Mark the resident entries whose flag is set dirty (host int32 per SPT id). */
int glod_cache_mark_dirty(glod_cache* c, const int32_t* flags, int32_t num_spts);
/* Disk mode (the reference's FileBacking, store.py:84-112):
 * the store stays in a .glod file (`fd` opened read-write, section_offset[k]
 * = byte offset of attribute section k).  Misses are pread() into pinned
 * bounce buffers and copied to HBM (prefetches while the GPU computes),
 * write-backs are copied back and pwrite()n before the next read.  Call
 * before the first step; the store view's section pointers are unused. */
int glod_cache_set_file(glod_cache* c, int32_t fd, const int64_t* section_offset);
/* Issue pending write-backs and (disk mode) complete them into the file;
 * reports the bytes read from / written to the file so far. */
int glod_cache_flush_io(glod_cache* c, int64_t* bytes_read, int64_t* bytes_written);
/* Resident entries in LRU order (front first), up to `capacity`. */
int glod_cache_entries(const glod_cache* c, int32_t* spt_id, double* cached_distance,
                       int64_t* prefix_len, uint64_t* block, int32_t* dirty, int64_t capacity);
/* K6 stable LSD radix sort of (key, int32 value) pairs by key bits
 * [begin_bit, end_bit) — the rasteriser's depth order and tile binning,
 * exported for direct use/testing.  keys/vals and their *_alt buffers:
 * [dev] length n; the sorted result ends in the alternates when
 * *result_in_alt == 1.  scratch: glod_sort_scratch_bytes(n) bytes. */
int64_t glod_sort_scratch_bytes(int64_t n);
int glod_sort_pairs_u64(uint64_t* keys, uint64_t* keys_alt, int32_t* vals, int32_t* vals_alt,
                        int64_t n, int32_t begin_bit, int32_t end_bit, void* scratch,
                        int64_t scratch_bytes, int32_t* result_in_alt, void* stream);
int glod_sort_pairs_u32(uint32_t* keys, uint32_t* keys_alt, int32_t* vals, int32_t* vals_alt,
                        int64_t n, int32_t begin_bit, int32_t end_bit, void* scratch,
                        int64_t scratch_bytes, int32_t* result_in_alt, void* stream);
/* Stream-ordered small device→host read-back into page-locked host memory,
 * written by a kernel through the mapped address (no copy engine, so it
 * never queues behind bulk D2H DMA).  The caller synchronises the stream
 * before reading host_pinned. */
int glod_readback(void* host_pinned, const void* src, int64_t bytes, void* stream);
/* Up to 8 such read-backs (4-byte aligned, multiples of 4 bytes) in one
 * kernel launch. */
int glod_readback_multi(int32_t n, void* const* host_pinned, const void* const* src, const int64_t* bytes,
                        void* stream);
/* The reverse: a stream-ordered small host→device upload read by a kernel
 * from page-locked memory (no copy-engine queueing behind the cache's bulk
 * prefetch DMA).  host_pinned must stay unchanged until the stream has run
 * the upload; pageable memory falls back to cudaMemcpyAsync. */
int glod_upload(void* dst, const void* host_pinned, int64_t bytes, void* stream);
/* Diagnostics: %globaltimer stamps (ns) of the last select launch's block 0
 * at its phase boundaries (start, flags, upper walks, passthrough walks,
 * bitmap counts, id lists, d_root/prefix); synchronises the device. */
int glod_debug_select_phases(int64_t* ns_out7);
/* Synchronous device→host copy (snapshots / tests). */
int glod_memcpy_d2h(void* dst, const void* src, int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* GLOD_B200_H */

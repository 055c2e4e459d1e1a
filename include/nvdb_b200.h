/*
 * nvdb_b200.h -- C ABI of the B200-native NeuralVDB hot path.
 *
 * Plain pointers and sizes only; every compute entry point takes a
 * cudaStream_t (as void*) and DEVICE pointers owned by the caller.  The
 * library never frees caller memory; the two handle types (netset, tree)
 * are library-owned, immutable after create and destroyed explicitly.
 *
 * Return value: 0 on success, a negative NVDB_E* code otherwise; the
 * message is available from nvdb_last_error() (thread-local).  No C++
 * exception crosses this boundary.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/svcodec/).
 */
#ifndef NVDB_B200_H
#define NVDB_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NVDB_API __attribute__((visibility("default")))
#else
#define NVDB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NVDB_OK 0
#define NVDB_EINVAL (-1)      /* bad argument  -> ValueError            */
#define NVDB_ECUDA (-2)       /* CUDA failure  -> RuntimeError          */
#define NVDB_EUNSUPPORTED (-3)/* shape not supported by this build       */
#define NVDB_ECORRUPT (-4)    /* inconsistent container -> SvcodecError */
#define NVDB_ENOMEM (-5)      /* workspace too small                     */

/* activation / head / net tag codes (neural.py:24-30, encoder.py:86) */
#define NVDB_ACT_RELU 0
#define NVDB_ACT_TANH 1
#define NVDB_ACT_SINE 2
#define NVDB_HEAD_LINEAR 0
#define NVDB_HEAD_LOGITS 1
#define NVDB_HEAD_BINARY 2
#define NVDB_TAG_L1 0
#define NVDB_TAG_TILE 1
#define NVDB_TAG_L0 2
#define NVDB_TAG_VOXEL 3

/* One coordinate network (MlpParams + FourierFeatures, neural.py:51-165).
 * HOST pointers; weights are the serialized (interleaved-feature) layout. */
typedef struct {
  int32_t m;           /* Fourier feature count (in_dim = 2m)          */
  int32_t depth;       /* hidden layers                                 */
  int32_t width;       /* hidden width                                  */
  int32_t out_dim;     /* 1 or 3                                        */
  int32_t activation;  /* NVDB_ACT_*                                    */
  int32_t head;        /* NVDB_HEAD_*                                   */
  float frequency;     /* sine frequency (omega)                        */
  float amplitude;     /* feature amplitude                             */
  const float* b2pi;   /* (3, m) float32 = (2*pi*B^T).astype(float32)   */
  const float* const* weights; /* depth+1 arrays W_l (out, in) row-major */
  const float* const* biases;  /* depth+1 arrays b_l (out,)              */
} nvdb_net_desc;

/* One subdomain expert (EncodedSubdomain, container.py:118-150). */
typedef struct {
  int32_t cell[3];
  int32_t net_index[4];   /* per tag l1/tile/l0/voxel: index into nets[] or -1 */
  double norm_origin[3];
  double norm_scale;
} nvdb_expert_desc;

typedef struct nvdb_netset nvdb_netset;
typedef struct nvdb_tree nvdb_tree;

NVDB_API const char* nvdb_last_error(void);
NVDB_API int nvdb_version(void);
/* number of kernels this library has launched in this process */
NVDB_API long long nvdb_launch_count(void);

/* -- networks ------------------------------------------------------------- */

/* Upload every expert's nets (replaces the per-call weight handling of
 * inference.eval_net, inference.py:23-26). */
NVDB_API int nvdb_netset_create(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                       int32_t nexperts, int32_t subdomain_size, int32_t halo, nvdb_netset** out);
/* Device bytes a netset of these nets needs, and its creation inside a
 * CALLER-OWNED device buffer: packed on the host, uploaded with an async copy
 * on `stream` (no host synchronisation, no cudaMalloc/cudaFree); destroy then
 * frees only the host handle.  The buffer must outlive the handle. */
NVDB_API int nvdb_netset_device_bytes(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                                      int32_t nexperts, int32_t subdomain_size, int32_t halo, size_t* bytes);
NVDB_API int nvdb_netset_create_at(const nvdb_net_desc* nets, int32_t nnets, const nvdb_expert_desc* experts,
                                   int32_t nexperts, int32_t subdomain_size, int32_t halo, void* device_mem,
                                   size_t device_bytes, void* stream, nvdb_netset** out);
NVDB_API int nvdb_netset_destroy(nvdb_netset* ns);

/* neural.forward_block (neural.py:527-550): raw outputs of net `net` at n
 * normalized float32 points pts (n,3); out (n, out_dim) float32. */
NVDB_API int nvdb_forward(const nvdb_netset* ns, int32_t net, const float* pts, int64_t n, float* out,
                 void* stream);

/* Workspace bytes needed by nvdb_eval_blended for n points. */
NVDB_API size_t nvdb_eval_workspace_bytes(const nvdb_netset* ns, int64_t n);

/* inference.blended_l1_probs / blended_l0_probs / blended_values
 * (inference.py:39-84, partition.py:180-256): gate-blended outputs at n
 * float64 index-space centres (n,3).  out (n, k) float64 (k = 3 for the l1
 * tag, else 1); covered (n,) uint8. */
NVDB_API int nvdb_eval_blended(const nvdb_netset* ns, int32_t tag, const double* centers, int64_t n,
                      double* out, uint8_t* covered, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Generic evaluation: point source x output selector. */
#define NVDB_SRC_NORM_F32 0   /* (n,3) float32 already-normalized inputs      */
#define NVDB_SRC_CENTER_F64 1 /* (n,3) float64 index-space centres            */
#define NVDB_SRC_COORD_I32 2  /* (n,3) int32 voxel coords, centre = c + 0.5   */
#define NVDB_SRC_LEAF_VOX 3   /* id = leaf*512 + voxel over (nl,3) int32 origins */
#define NVDB_SRC_L1_SLOT 4    /* id = node*4096 + slot over (n1,3) int32 origins  */
#define NVDB_OUT_RAW 0        /* raw head outputs (single net)                */
#define NVDB_OUT_PROBS 1      /* blended float64 (n,k) + covered u8           */
#define NVDB_OUT_L1CLASS 2    /* u8 argmax of blended probs, uncovered -> 2   */
#define NVDB_OUT_L0ACTIVE 3   /* u8 covered && p > 0.5                        */
#define NVDB_OUT_VALUE 4      /* f32 covered ? clip?(v)*scale : background    */

typedef struct {
  int32_t out_mode;
  float* raw;
  double* probs;
  uint8_t* u8;
  float* f32;
  double value_scale;
  float background;
  int32_t clip;
} nvdb_eval_out;

/* The fused evaluator behind every decode stage (decoder.py:110-196) and
 * the blended seams: point ids 0..n-1 (source id gather[i] when gather is
 * non-null), outputs written at index i.  Workspace: nvdb_eval_workspace_bytes.
 * Calls above 2^30 points run as consecutive 2^30-point chunks (the workspace
 * covers one chunk); the counted form below takes at most 2^30 points. */
NVDB_API int nvdb_eval(const nvdb_netset* ns, int32_t tag, int32_t src_kind, const void* src,
                       const int64_t* gather, int64_t n, const nvdb_eval_out* out, void* workspace,
                       size_t workspace_bytes, void* stream);
/* nvdb_eval over the first *count_dev points (device int64, e.g. written by
 * nvdb_select_u8) of a buffer of `capacity`: the count never visits the host,
 * so a decode chains select -> eval without a stream synchronisation.  The
 * workspace is sized for `capacity`; outputs past the count are untouched. */
NVDB_API int nvdb_eval_counted(const nvdb_netset* ns, int32_t tag, int32_t src_kind, const void* src,
                               const int64_t* gather, int64_t capacity, const int64_t* count_dev,
                               const nvdb_eval_out* out, void* workspace, size_t workspace_bytes, void* stream);

/* -- decode helpers (decoder.py:101-211) ------------------------------------ */

/* ids of entries equal to `value` (ascending) and their count (device int64). */
NVDB_API size_t nvdb_select_workspace_bytes(int64_t n);
NVDB_API int nvdb_select_u8(const uint8_t* v, int64_t n, uint8_t value, int64_t* ids, int64_t* count,
                            void* workspace, size_t workspace_bytes, void* stream);
/* level-1 patches then inactive tile values where class == 2 (decoder.py:114-134) */
NVDB_API int nvdb_l1_apply(uint8_t* cls, float* tiles, int64_t nslots, const int64_t* patch_slot,
                           const uint8_t* patch_cls, int64_t npatch, const int64_t* tile_slot,
                           const float* tile_value, int64_t ntile, void* stream);
NVDB_API int nvdb_scatter_f32(float* dst, const int64_t* ids, const float* vals, int64_t n, void* stream);
/* dst[ids[i]] = vals[i] for i < *count_dev (device int64, <= capacity). */
NVDB_API int nvdb_scatter_f32_counted(float* dst, const int64_t* ids, const float* vals, int64_t capacity,
                                      const int64_t* count_dev, void* stream);
/* as nvdb_scatter_f32_counted, skipping ids with skip[id] != 0: the voxel
 * regressor's values of one leaf range after nvdb_leaf_finalize_counted ran
 * without them (patched voxels keep their patch value; decoder.py:191-196) */
NVDB_API int nvdb_scatter_f32_unpatched_counted(float* dst, const int64_t* ids, const float* vals, int64_t capacity,
                                                const int64_t* count_dev, const uint8_t* skip, void* stream);
/* leaf origins of child slots (node*4096+slot, node order x ascending slot)
 * and the slot -> leaf index map (-1 elsewhere) (decoder.py:146-151) */
/* Level-1 slot (node * 4096 + idx1, -1 outside every node) and idx0 of
 * int32 coordinates (n,3), the node found through a dense int32 table over
 * the bounding box [lut_lo, lut_lo + lut_span) of the level-1 origins >> 7
 * (node index in sorted-origin order or -1); lut_lo / lut_span are HOST
 * int32[3].  err (nullable, DEVICE) is set to 1 when a coordinate lies in no
 * node.  vox nullable. */
NVDB_API int nvdb_node_slots(const int32_t* lut, const int32_t* lut_lo, const int32_t* lut_span,
                             const int32_t* coords, int64_t n, int64_t* slot, int32_t* vox, int32_t* err,
                             void* stream);
NVDB_API int nvdb_leaf_list(const int64_t* child_slots, int64_t nl, const int32_t* node_origins,
                            int64_t nslots, int32_t* leaf_origins, int32_t* leaf_of_slot, void* stream);
/* level-0 patches on the active mask; *err = 1 if a patch has no leaf (decoder.py:168-179) */
NVDB_API int nvdb_l0_apply(uint8_t* active, const int64_t* patch_slot, const int32_t* patch_vox,
                           const uint8_t* patch_active, int64_t npatch, const int32_t* leaf_of_slot,
                           int32_t* err, void* stream);
/* leaf values: background, regressed active voxels, patch values, negative
 * fill of inactive voxels; packed active words; optional patched flags
 * (decoder.py:182-210) */
NVDB_API int nvdb_leaf_finalize(int64_t nl, const uint8_t* active, const int64_t* act_ids,
                                const float* act_vals, int64_t nact, const int64_t* patch_slot,
                                const int32_t* patch_vox, const uint8_t* patch_active,
                                const float* patch_value, int64_t npatch, const int64_t* neg_slot,
                                const uint64_t* neg_bits, int64_t nneg, const int32_t* leaf_of_slot,
                                float background, float neg_value, float* values,
                                uint64_t* active_words, uint8_t* patched, void* stream);
/* nvdb_leaf_finalize with the regressed-voxel count on the device
 * (*nact_dev <= act_capacity, from nvdb_select_u8): no host round trip. */
NVDB_API int nvdb_leaf_finalize_counted(int64_t nl, const uint8_t* active, const int64_t* act_ids,
                                        const float* act_vals, int64_t act_capacity, const int64_t* nact_dev,
                                        const int64_t* patch_slot, const int32_t* patch_vox,
                                        const uint8_t* patch_active, const float* patch_value, int64_t npatch,
                                        const int64_t* neg_slot, const uint64_t* neg_bits, int64_t nneg,
                                        const int32_t* leaf_of_slot, float background, float neg_value,
                                        float* values, uint64_t* active_words, uint8_t* patched, void* stream);
/* words[w] bit j = (v[64w + j] == value) */
NVDB_API int nvdb_pack_eq(const uint8_t* v, int64_t nwords, uint8_t value, uint64_t* words, void* stream);

/* -- upper-tree lookup ----------------------------------------------------- */

/* Flattened [Hash,5,4,3] tree (grid.py:248-390).  HOST arrays:
 *   root keys (nr,3) + per root: l2 node index or -1, tile value, tile active
 *   l2 nodes (n2): origin (n2,3); child/active bit words (n2, 512) uint64;
 *                  tiles (n2, 32768) float32
 *   l1 nodes (n1): origin (n1,3); child/active (n1, 64) uint64; tiles (n1, 4096)
 *   leaves  (nl): active (nl, 8) uint64; values (nl, 512) float32
 * Children are implied by mask order: the k-th set child bit of l2 node i is
 * l1 node l2_child_base[i] + k, likewise l1 -> leaves. */
typedef struct {
  float background;
  int32_t nroots, n2, n1, nl;
  const int32_t* root_keys;        /* (nroots,3) */
  const int32_t* root_l2;          /* (nroots) l2 index or -1 (tile) */
  const float* root_tile_value;    /* (nroots) */
  const uint8_t* root_tile_active; /* (nroots) */
  const uint64_t* l2_child;        /* (n2,512) */
  const uint64_t* l2_active;       /* (n2,512) */
  const float* l2_tiles;           /* (n2,32768) */
  const int32_t* l2_child_base;    /* (n2) */
  const uint64_t* l1_child;        /* (n1,64) */
  const uint64_t* l1_active;       /* (n1,64) */
  const float* l1_tiles;           /* (n1,4096) */
  const int32_t* l1_child_base;    /* (n1) */
  const uint64_t* leaf_active;     /* (nl,8) */
  const float* leaf_values;        /* (nl,512) */
  const uint64_t* leaf_patched;    /* (nl,8) or NULL: voxels holding exact patch values */
} nvdb_tree_desc;
/* (all tree_desc arrays may be host or device memory) */

NVDB_API int nvdb_tree_create(const nvdb_tree_desc* desc, nvdb_tree** out);
NVDB_API int nvdb_tree_destroy(nvdb_tree* tree);

/* VdbGrid.get_values(coords, with_kind=True) (grid.py:310-390): device
 * int32 coords (n,3) -> value f32, active u8, kind u8 (0 none,1 tile,2 leaf);
 * leaf (n) int32 leaf index or -1 (nullable). */
NVDB_API int nvdb_lookup(const nvdb_tree* tree, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                uint8_t* kind, int32_t* leaf, void* stream);

/* nvdb_lookup fused with the query's neural-row selection (decoder.py:243):
 * value/active/kind as nvdb_lookup, and the rows with active && kind == 2
 * appended to rows (capacity n, int64 row ids, order not deterministic) with
 * their number in *count (device int64).  Rows whose voxel holds an exact
 * patch already have their final value and are counted in *npatched
 * (device int64) instead: regressor evaluations = *count + *npatched.
 * coords/value 16-byte and active/kind 4-byte aligned. */
NVDB_API int nvdb_lookup_rows(const nvdb_tree* tree, const int32_t* coords, int64_t n, float* value, uint8_t* active,
                              uint8_t* kind, int64_t* rows, int64_t* count, int64_t* npatched, void* stream);

/* HybridGrid.query (decoder.py:239-264) pieces: flag rows with active &&
 * kind == 2, then write regressed values (patched voxels keep their exact
 * stored value from the tree) back to those rows. */
NVDB_API int nvdb_neural_rows(const uint8_t* active, const uint8_t* kind, int64_t n, uint8_t* flag, void* stream);
NVDB_API int nvdb_query_finalize(const int64_t* rows, int64_t nrows, const float* regressed,
                                 const int32_t* coords, const int32_t* leaf, const nvdb_tree* tree,
                                 float* value, void* stream);
/* nvdb_query_finalize over the first *nrows_dev rows (device int64) of `capacity`. */
NVDB_API int nvdb_query_finalize_counted(const int64_t* rows, int64_t capacity, const int64_t* nrows_dev,
                                         const float* regressed, const int32_t* coords, const int32_t* leaf,
                                         const nvdb_tree* tree, float* value, void* stream);

/* -- NVGR emission (gridfile.py:43-76) ------------------ */
/* Leaf records (origin i32x3 | packbits-little active mask 64 B | 512 f32
 * values, 2124 B) of a dense-leaf decode, leaf r written at out + rec_off[r]
 * (byte offsets into the NVGR stream, any alignment).  DEVICE pointers. */
NVDB_API int nvdb_nvgr_leaf_records(const int32_t* leaf_origins, const uint64_t* active_words,
                                    const float* values, int64_t nleaves, const int64_t* rec_off, uint8_t* out,
                                    void* stream);
/* Level-1 node records (origin | child mask 512 B (class 0) | active mask
 * 512 B (class 1) | 4096 f32 tiles, 17420 B) from the decode's per-slot
 * classes and tiles (node order of node_origins).  DEVICE pointers. */
NVDB_API int nvdb_nvgr_l1_records(const int32_t* node_origins, const uint8_t* l1_class, const float* tiles,
                                  int64_t nnodes, const int64_t* rec_off, uint8_t* out, void* stream);

/* -- verification metrics (metrics.py:116-230) --------- */
/* One pass of grid A against grid B: enumerates A's leaf voxels (origins in
 * A's tree order, DEVICE int32 (nl,3)) and A's tile extents (host-compacted
 * list: origin, extent 8|128, value, active, prefix of extent^3 (ntiles+1);
 * DEVICE), resolving each coordinate in B.  Adds 8 double sums per block to
 * `partials` (nvdb_metric_partials() blocks x 8, DEVICE, zeroed here):
 * |act A|, |act A & act B|, |occ A|, |occ A & occ B|, sum over act A & act B
 * of (vA - vB)^2, sum over act A & !act B of (vA - bg_B)^2, surface points
 * of A, sum of |trilinear_B| at them (want_mcd != 0). */
NVDB_API size_t nvdb_metric_partials(void);
NVDB_API int nvdb_metric_pass(const nvdb_tree* a, const int32_t* a_leaf_origins, const nvdb_tree* b,
                              const int32_t* tile_origin, const int32_t* tile_extent, const float* tile_value,
                              const uint8_t* tile_active, const int64_t* tile_first, int64_t ntiles, int32_t sdf,
                              int32_t want_mcd, double* partials, void* stream);

/* -- training (encoder.train_network, encoder.py:330-371) -------------------- */

#define NVDB_LOSS_MSE 0
#define NVDB_LOSS_CE 1
#define NVDB_LOSS_BCE 2

typedef struct nvdb_trainer nvdb_trainer;

typedef struct {
  nvdb_net_desc net;        /* initial (cold or warm) weights, HOST            */
  int32_t loss_kind;        /* NVDB_LOSS_*                                      */
  int64_t n;                /* training points                                  */
  const float* inputs;      /* DEVICE (n,3) float32 normalized inputs           */
  const float* targets;     /* DEVICE (n,) float32 targets (labels as floats)   */
  int32_t batch;            /* cfg.batch_size                                   */
  int32_t sampled;          /* 1: per-epoch Sampler draws (n > batch and not full-batch) */
  int32_t sample_interval;  /* cfg.sample_interval (1 supported)                */
  int32_t max_epochs;
  const float* lr;          /* HOST (max_epochs) float32(lr_at(schedule, e))    */
  const float* c1;          /* HOST (max_epochs) float32(1 - 0.9^(e+1))         */
  const float* c2;          /* HOST (max_epochs) float32(1 - 0.999^(e+1))       */
  const uint64_t* seed_words; /* HOST (max_epochs,4) SeedSequence((seed,0,e)).generate_state(4,u64) */
  double target_loss;       /* early stop when the pre-update epoch loss < target */
  int32_t shard_rank;       /* data parallel: this rank's contiguous share of the batch tiles */
  int32_t shard_count;      /* ranks (<= 1: the whole batch)                                */
  int32_t path;             /* 0 auto; 1 fused kernels (weights resident in shared memory,
                               hidden width <= 128); 2 layer-streamed kernels (any shape up
                               to width 256, 2m 1024; the auto choice when 1 does not fit) */
} nvdb_train_desc;

NVDB_API int nvdb_trainer_create(const nvdb_train_desc* desc, nvdb_trainer** out);
/* Does not synchronize: the trainer's device blocks go to a per-device cache
 * with an event recorded after its last enqueued work, and the next trainer
 * created on that device waits for the event before reusing them. */
NVDB_API int nvdb_trainer_destroy(nvdb_trainer* tr);
/* Release the trainer block cache of every device; returns the bytes freed. */
NVDB_API size_t nvdb_trim(void);
/* enqueue `epochs` epochs (sampler -> fwd/dgrad -> wgrad -> Adam); epochs
 * after the early stop are no-ops on the device; enqueueing more than
 * max_epochs epochs in total returns NVDB_EINVAL */
NVDB_API int nvdb_trainer_run(nvdb_trainer* tr, int32_t epochs, void* stream);
/* Bound the CTAs (one per SM) this trainer's epoch kernels launch with, so
 * several trainers on separate streams train concurrently on disjoint SMs
 * (the survey's grouped launch of a container's nets, §7 hard part 4).
 * 0 = every SM; never more than at creation.  Takes effect at the next
 * enqueued epoch; the gradient summation order follows the CTA count. */
NVDB_API int nvdb_trainer_set_ctas(nvdb_trainer* tr, int32_t ctas);
/* one epoch split for data parallelism: phase 1 = sampler (the first call
 * presamples every epoch), fwd/dgrad, wgrad, partial reduction into the
 * packed buffer; phase 2 = Adam, early stop, epoch advance.  Between them the
 * caller all-reduces (sum) the packed buffer across ranks -- ONE collective
 * per epoch (NCCL over NVLink).  Phase launches read the epoch from device
 * memory, so one captured (phase 1, all-reduce, phase 2) graph can be
 * replayed for every epoch; replays after the early stop are no-ops. */
NVDB_API int nvdb_trainer_phase(nvdb_trainer* tr, int32_t phase, void* stream);
/* packed buffer of *nfloats = nparams + 2 floats: the gradient sums, then the
 * batch-loss sum as an f32 (hi, lo) pair that phase 2 recombines in f64 */
NVDB_API int nvdb_trainer_packed(nvdb_trainer* tr, float** buf, int64_t* nfloats);
/* the gradient (nparams floats, the head of the packed buffer) and this
 * rank's local batch-loss sum (informational; phase 2 reads the packed pair) */
NVDB_API int nvdb_trainer_buffers(nvdb_trainer* tr, float** grad, int64_t* nparams, double** loss);
/* synchronous: epochs run so far, stop flag, per-epoch losses (HOST out) */
NVDB_API int nvdb_trainer_status(const nvdb_trainer* tr, int32_t* epochs_done, int32_t* stopped,
                                 double* losses, int32_t nlosses);
/* encoder.Sampler.indices (encoder.py:257-267, sample_interval 1): `batch`
 * numpy-exact draws in [0, n) from PCG64 seeded with the 4 HOST words of
 * SeedSequence((seed, 0, epoch)).generate_state(4, uint64); idx DEVICE. */
NVDB_API int nvdb_sample_indices(uint64_t n, int64_t batch, const uint64_t* words, int64_t* idx, void* stream);
/* encoder.Sampler.indices with sample_interval > 1 (encoder.py:260-267): the
 * working subset of interval*batch draws in [0, n) from the HOST words of
 * SeedSequence((seed, 1, epoch // interval)), then `batch` draws in
 * [0, interval*batch) from SeedSequence((seed, 2, epoch)) mapped through it;
 * idx DEVICE.  nvdb_train_desc.seed_words holds, for sample_interval > 1, the
 * (seed, 2, epoch) words of every epoch followed by the (seed, 1, chunk)
 * words of every chunk. */
NVDB_API int nvdb_sample_indices_subset(uint64_t n, int64_t batch, int32_t interval, const uint64_t* words_epoch,
                                        const uint64_t* words_chunk, int64_t* idx, void* stream);
/* fp32 master weights into HOST arrays shaped like nvdb_net_desc */
NVDB_API int nvdb_trainer_weights(const nvdb_trainer* tr, float* const* weights, float* const* biases);

/* -- synthetic inputs ------------------------------------ */

/* procgen.FbmSpec: value-noise fBm density over the index box [lo, hi]
 * (inclusive; the reference's domain hi minus one) */
typedef struct {
  int32_t octaves;
  double lacunarity, gain, base_frequency;
  uint64_t seed;
  int32_t lo[3], hi[3];
  double threshold, voxel_size;
} nvdb_fbm_desc;

/* gen_fbm_density (procgen.py:283-309) per leaf block: for the nblocks leaf
 * origins (int3, DEVICE) write the 512 voxel values (f32: fbm where active,
 * else 0) and active flags, and set keep[b] = 1 (int32, DEVICE, caller
 * zeroed) for blocks with an active voxel.  Bit-exact with the reference. */
NVDB_API int nvdb_fbm_leaves(const nvdb_fbm_desc* spec, const int32_t* origins, int64_t nblocks, float* values,
                             uint8_t* active, int32_t* keep, void* stream);

/* -- diagnostics ------------------------------------------------------------ */

/* One 128xN tcgen05 MMA over nk K-steps from caller-laid-out shared-memory
 * images (used by the descriptor-layout unit tests). Device pointers. */
NVDB_API int nvdb_selftest_umma(const void* a_img, uint32_t a_bytes, const void* b_img, uint32_t b_bytes,
                       int32_t n, int32_t nk, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_step,
                       uint32_t b_lbo, uint32_t b_sbo, uint32_t b_step, int32_t a_mn, int32_t b_mn,
                       float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NVDB_B200_H */

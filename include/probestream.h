/*
 * probestream.h -- C ABI of the B200-native probe-streaming hot path.
 *
 * Drop-in boundary for the reference's Python entry points
 * (/root/reference/pkg/src/probestream/).  Every entry point takes plain
 * device pointers, sizes and a cudaStream_t passed as `void *`; none
 * allocates (scratch comes from the caller, sized by the *_workspace_bytes
 * queries) and none synchronises the stream.  All work is stream-ordered.
 *
 * Status codes map 1:1 onto the reference's exception classes; the Python
 * shim (paper_2103_05875_b200/_native.py) re-raises the same classes.
 * Validation the reference performs before mutating state happens here
 * before any launch.
 *
 * Texel formats (volume.py:147-154): colour = uint32 (H, W) with R/G/B in
 * bits 0-9/10-19/20-29; visibility = uint16 (H, W, 2) raw half bits.
 * Probe p's block sits at block row p / probes_per_row, block column
 * p % probes_per_row (volume.py:198-203).
 */
#ifndef PROBESTREAM_H
#define PROBESTREAM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_ABI_VERSION 10

/* status codes */
#define PS_OK 0
#define PS_ERR_VALUE (-1)         /* ValueError (packing.py:80, :120, :140)            */
#define PS_ERR_LAYOUT (-2)        /* LayoutMismatchError(ValueError) (selection.py:25)  */
#define PS_ERR_SLOT_OVERFLOW (-3) /* SlotOverflowError(RuntimeError) (packing.py:227)   */
#define PS_ERR_INDEX (-4)         /* IndexError (volume.py:199, packing.py:273)         */
#define PS_ERR_CUDA (-5)          /* RuntimeError: CUDA launch / runtime failure        */
#define PS_ERR_WORKSPACE (-6)     /* ValueError: caller workspace too small             */

#define PS_KIND_COLOR 0
#define PS_KIND_VISIBILITY 1

#define PS_SHADOW_NONE 0
#define PS_SHADOW_RAYS 1
#define PS_SHADOW_MAP 2

/* device-side status word bits (written by kernels, read by the shim) */
#define PS_DEV_SLOT_OVERFLOW 1u   /* selection larger than slot_count, nothing mutated */
#define PS_DEV_INDEX 2u           /* id outside [0, probe_count)                       */

/* thread-local message for the last non-zero status */
const char *ps_last_error(void);
int ps_abi_version(void);
/* number of SMs of the current device (grid sizing helper for the shim) */
int ps_device_sm_count(void);

/* ---------------------------------------------------------------------------
 * Stage (4): plane packing.
 * ------------------------------------------------------------------------- */

/* pack_color (packing.py:73-89): texels uint32 (h, w) with row stride
 * `row_stride` elements -> planes uint16 (3, h, w) contiguous. */
int ps_pack_color(const uint32_t *texels, int64_t h, int64_t w, int64_t row_stride,
                  uint16_t *planes, void *stream);

/* widened_width (packing.py:105-109) = ceil(4w/3); -1 if w < 0 */
int64_t ps_widened_width(int64_t w);

/* pack_visibility (packing.py:112-133): texels uint16 (h, w, 2) with row
 * stride `row_stride` texels -> planes uint8 (3, h, ceil(4w/3)) contiguous. */
int ps_pack_visibility(const uint16_t *texels, int64_t h, int64_t w, int64_t row_stride,
                       uint8_t *planes, void *stream);

/* unpack_* (packing.py:92-99, :136-151): client-side inverses, used as
 * round-trip verifiers. */
int ps_unpack_color(const uint16_t *planes, int64_t h, int64_t w, uint32_t *texels,
                    void *stream);
int ps_unpack_visibility(const uint8_t *planes, int64_t h, int64_t w, uint16_t *texels,
                         void *stream);

/* Temporal delta (codec.py:207-215 residual, :250-272 SKIP rule) over plane
 * sets of `elem_bytes` (2 = colour uint16, 1 = visibility uint8) elements,
 * shape (3, h, w).  residual = (cur - prev) mod 2^bits; skip is uint8
 * (3, ceil(h/16), ceil(w/16)), 1 where the clipped 16x16 block is
 * bit-identical.  prev == NULL is a key frame: residual untouched, skip 0. */
int ps_temporal_delta(int elem_bytes, const void *cur, const void *prev, int64_t h,
                      int64_t w, void *residual, uint8_t *skip, void *stream);

/* Fused pack + temporal delta over a whole update atlas: writes planes_cur,
 * residual (vs planes_prev) and skip in one pass.  planes_prev == NULL is a
 * key frame (residual untouched, skip 0); so is a non-zero *key_dev (optional
 * device flag, lets a captured CUDA graph decide per replay). */
int ps_pack_delta(int kind, const void *texels, int64_t h, int64_t w, int64_t row_stride,
                  void *planes_cur, const void *planes_prev, void *residual,
                  uint8_t *skip, const int32_t *key_dev, void *stream);

/* LPF1 frame encoding (codec.py:335-366), bit-exact: planes (3, h, w) of
 * elem_bytes (2 colour, 1 visibility) elements; reference == NULL encodes a
 * key frame (left-neighbour intra prediction), else a P-frame against the
 * reference planes (SKIP / DELTA / RAW blocks).  Writes header + payload +
 * CRC32 into `out` (capacity from ps_encode_frame_capacity) and the frame
 * length into the device scalar *frame_len. */
int64_t ps_encode_frame_capacity(int64_t h, int64_t w, int elem_bytes);
size_t ps_encode_workspace_bytes(int64_t h, int64_t w, int elem_bytes);
int ps_encode_frame(int elem_bytes, const void *planes, const void *reference, int64_t h,
                    int64_t w, uint32_t stream_id, uint32_t frame_seq, uint8_t *out,
                    int64_t out_capacity, int64_t *frame_len, void *workspace,
                    size_t workspace_bytes, void *stream);

/* Client side (verifier of the server path): LPF1 decode (codec.py:369-395)
 * of a frame whose bytes are on the device (`frame` points at the header,
 * payload_len from the header); reference planes for P-frames, NULL for a
 * key frame.  Structural errors set bits in *status_dev (1 corrupt frame, 2
 * malformed entropy stream); nothing is raised from the device. */
size_t ps_decode_workspace_bytes(int64_t h, int64_t w);
int ps_decode_frame(int elem_bytes, const uint8_t *frame, int64_t payload_len,
                    const void *reference, int64_t h, int64_t w, void *planes_out,
                    uint32_t *status_dev, void *workspace, size_t workspace_bytes, void *stream);
/* apply_update_entries (packing.py:341-350): slot cores into probe blocks of
 * `atlas` with the guard band rebuilt. */
int ps_apply_entries(int kind, const void *update_texels, int64_t update_row_stride,
                     int64_t slots_per_row, const int64_t *entries, const int64_t *entry_count,
                     int64_t max_entries, void *atlas, int64_t probes_per_row, void *stream);

/* ---------------------------------------------------------------------------
 * Stage (3): change detection and compaction (selection.py:284-323).
 * ------------------------------------------------------------------------- */

/* threshold handling mirrors the reference's numpy promotion:
 *   threshold <= 0                  -> exact bit compare of the full block;
 *   colour, threshold > 0 (or NaN)  -> max channel |delta| > threshold;
 *   visibility, threshold > 0/NaN   -> |f32(a)-f32(b)| > thr OR (NaN delta and
 *                                      bits differ); thr is compared as float32
 *                                      unless threshold_is_f64 (a numpy float64
 *                                      scalar in the caller). */
size_t ps_detect_workspace_bytes(int64_t probe_count);
int ps_detect_changed(int kind, const void *rendered, const void *last_sent,
                      int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                      const uint8_t *active, double threshold, int threshold_is_f64,
                      uint32_t *changed_bits, int64_t *out_ids, int64_t *out_count,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Same, restricted to probes [probe_begin, probe_end) (a z-slab of a sharded
 * volume): only those bits can be set; only the block rows covering the range
 * are read. */
int ps_detect_changed_range(int kind, const void *rendered, const void *last_sent,
                            int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                            int64_t probe_begin, int64_t probe_end, const uint8_t *active,
                            double threshold, int threshold_is_f64, uint32_t *changed_bits,
                            int64_t *out_ids, int64_t *out_count, void *workspace,
                            size_t workspace_bytes, void *stream);

/* Bitmap <-> id list helpers.  ids_to_bits ORs ids[0..n) (n read from
 * n_dev when non-NULL, else n_host) into bits (caller zeroes) and sets
 * PS_DEV_INDEX in *status_dev for ids outside [0, probe_count).
 * bits_to_ids writes ascending ids (flatnonzero) and the count. */
int ps_ids_to_bits(const int64_t *ids, const int64_t *n_dev, int64_t n_host,
                   int64_t probe_count, uint32_t *bits, uint32_t *status_dev, void *stream);
size_t ps_compact_workspace_bytes(int64_t probe_count);
int ps_bits_to_ids(const uint32_t *bits, int64_t probe_count, int64_t *out_ids,
                   int64_t *out_count, void *workspace, size_t workspace_bytes, void *stream);

/* Potentially visible probes (selection.py:384-407) over a triangle scene:
 * ray_dirs (ray_count, 3) float64 from pvs_rays (frustum grid + fibonacci
 * sphere), camera = pose.position, volume_origin / volume_spacing: HOST
 * pointers to 3 doubles each; vertices (T, 3, 3) float64 on the device
 * (the BVH's source triangles, world frame), BVH as built by
 * ps_bvh_build_wide with its frame header before node 0 (see there).  Writes
 * the active-masked cage bitmap and (optionally) ascending ids + count. */
size_t ps_pvs_workspace_bytes(int64_t probe_count);
int ps_pvs(const float *nodes, int32_t bvh_width, const float *tris, const double *vertices,
           const double *ray_dirs, int64_t ray_count, const double *camera, int32_t nx, int32_t ny,
           int32_t nz, const double *volume_origin, const double *volume_spacing,
           const uint8_t *active, uint32_t *mask_bits, int64_t *out_ids, int64_t *out_count,
           void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Stage (3) tail: budgeted selection (selection.py:413-437).
 * candidates = changed & pvs & active (bitmaps; pvs_bits NULL = all), ordered
 * by staleness (current_seq - last_sent_seq[p]) descending then id
 * ascending, truncated with python slice semantics when has_budget.
 * ordered = 0 without a budget returns the same set in ascending id order
 * (no sort): what the slot assignment consumes, which orders by id itself.
 * ------------------------------------------------------------------------- */
size_t ps_select_workspace_bytes(int64_t probe_count);
int ps_select(const uint32_t *changed_bits, const uint32_t *pvs_bits, const uint8_t *active,
              const int64_t *last_sent_seq, int64_t current_seq, int64_t probe_count,
              int has_budget, int64_t budget, int ordered, int64_t *out_ids,
              int64_t *out_count, void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Stage (4): update-atlas slot cache (packing.py:243-317) and build
 * (packing.py:320-338).  Slot state lives in device memory:
 *   probe_slot int32[probe_count] (-1 = none), slot_probe int32[slot_count],
 *   last_selected int64[probe_count], meta int64[4] = {tick, used, -, -}.
 * ------------------------------------------------------------------------- */
size_t ps_assign_workspace_bytes(int64_t probe_count, int64_t slot_count);
/* selected ids (any order, duplicates allowed): n from n_dev if non-NULL. On
 * overflow nothing is mutated, *status_dev |= PS_DEV_SLOT_OVERFLOW and
 * entry_count = 0.  entries = (slot, probe) int64 pairs sorted by slot. */
int ps_assign_slots(const int64_t *selected, const int64_t *n_dev, int64_t n_host,
                    int64_t probe_count, int64_t slot_count, int32_t *probe_slot,
                    int32_t *slot_probe, int64_t *last_selected, int64_t *meta,
                    int64_t *entries, int64_t *entry_count, uint32_t *status_dev,
                    void *workspace, size_t workspace_bytes, void *stream);

/* The same state machine straight from a selection BITMAP (bit p = probe p
 * selected; ANDed with pvs_bits when non-NULL), for slot_count >=
 * probe_count, where no eviction is reachable: two single-pass kernels
 * (decoupled look-back scans) instead of ps_assign_slots' id-list chain.
 * Writes probe_slot / slot_probe / last_selected / meta exactly as
 * ps_assign_slots, entries + entry_count, plan int64[8] (the per-call plan:
 * selected, new, taken-free, 0, 0, old used, tick) and, when non-NULL,
 * *sel_count.  PS_ERR_VALUE when slot_count < probe_count. */
size_t ps_assign_bits_workspace_bytes(int64_t probe_count, int64_t slot_count);
int ps_assign_slots_bits(const uint32_t *sel_bits, const uint32_t *pvs_bits, int64_t probe_count,
                         int64_t slot_count, int32_t *probe_slot, int32_t *slot_probe,
                         int64_t *last_selected, int64_t *meta, int64_t *entries,
                         int64_t *entry_count, int64_t *plan, int64_t *sel_count,
                         void *workspace, size_t workspace_bytes, void *stream);

/* Copy each entry's stripped core (block[1:-1,1:-1]) into its slot region of
 * update_texels (packing.py:335-337).  Optional commit: when
 * last_sent != NULL also copies the full block into last_sent and stamps
 * last_sent_seq[p] = current_seq (or *current_seq_dev when non-NULL).  Work
 * is bounded by *entry_count (device). */
int ps_build_update(int kind, const void *source, int64_t probe_count,
                    int64_t probes_per_row, const int64_t *entries,
                    const int64_t *entry_count, int64_t max_entries, int64_t slots_per_row,
                    void *update_texels, int64_t update_row_stride, void *last_sent,
                    int64_t *last_sent_seq, int64_t current_seq,
                    const int64_t *current_seq_dev, void *stream);

/* Slab-sharded build (multi-GPU, single encoder stream).  Every rank runs
 * the same selection + slot assignment; a rank then
 *   - copies the core of each entry whose probe lies in [probe_begin,
 *     probe_end) into `payload` at index (probe - probe_begin) (core_side^2
 *     texels per probe), commits the full block into last_sent (if non-NULL),
 *   - stamps last_sent_seq[p] = current_seq for EVERY entry (replicated state).
 * The encoder rank gathers the payloads of all ranks and imports them:
 *   update_texels[slot] = payload_r[(probe - rank_begin[r])] with r the rank
 *   whose [rank_begin[r], rank_begin[r+1]) holds the probe; payload_r sits at
 *   payloads + r * payload_stride probes. */
int ps_export_tiles(int kind, const void *source, int64_t probe_count, int64_t probes_per_row,
                    const int64_t *entries, const int64_t *entry_count, int64_t max_entries,
                    int64_t probe_begin, int64_t probe_end, void *payload, void *last_sent,
                    int64_t *last_sent_seq, int64_t current_seq,
                    const int64_t *current_seq_dev, void *stream);
int ps_import_tiles(int kind, const void *payloads, int64_t payload_stride,
                    const int64_t *rank_begin, int32_t world, const int64_t *entries,
                    const int64_t *entry_count, int64_t max_entries, int64_t slots_per_row,
                    void *update_texels, int64_t update_row_stride, void *stream);

/* Peer-memory exchanges of the slab-sharded frame (csrc/ps_peer.cu, new:
 * the reference has no multi-GPU path).
 *   ps_detect_changed_bcast: as ps_detect_changed_range, but every changed
 *     word is ORed (system-scope atomics) into each of the ndst bitmaps in
 *     dst_bits (a device array of device pointers, peers' mapped bitmaps
 *     included); the caller zeroes the bitmaps between frames.
 *   ps_export_tiles_peer: copies the cores of the selected probes inside
 *     [probe_begin, probe_end) into the slots of dst_update_texels (the
 *     encoder rank's update atlas, mapped from another process), commits
 *     them into last_sent and stamps last_sent_seq for every entry.
 *   ps_peer_signal: stores (value or *value_dev) + add into each *flags[i]
 *     with system-scope release semantics after a system fence;
 *     ps_peer_wait: spins until every flags[i] >= that value (acquire); with
 *     a non-null error word (host-mapped pinned int32) and timeout_ns > 0 the
 *     spin is bounded: on expiry it stores (flag index + 1) into *error and
 *     returns, so a dead peer cannot hang the survivors inside a kernel or a
 *     graph replay.  ps_peer_status returns PS_ERR_CUDA (with the message in
 *     ps_last_error) once *error is set, PS_OK otherwise; it reads host
 *     memory only and does not synchronise.
 *   ps_ipc_export / ps_ipc_open: CUDA IPC handle (ps_ipc_handle_bytes bytes)
 *     and offset for any device pointer; opening maps it in this process
 *     (cached per allocation). */
int ps_detect_changed_bcast(int kind, const void *rendered, const void *last_sent,
                            int64_t probe_count, int64_t probes_per_row, int64_t block_rows,
                            int64_t probe_begin, int64_t probe_end, const uint8_t *active,
                            double threshold, int threshold_is_f64, uint32_t *const *dst_bits,
                            int ndst, void *stream);
int ps_export_tiles_peer(int kind, const void *source, int64_t probe_count,
                         int64_t probes_per_row, const int64_t *entries,
                         const int64_t *entry_count, int64_t max_entries, int64_t probe_begin,
                         int64_t probe_end, int64_t slots_per_row, void *dst_update_texels,
                         int64_t dst_row_stride, void *last_sent, int64_t *last_sent_seq,
                         int64_t current_seq, const int64_t *current_seq_dev, void *stream);
int ps_peer_signal(int64_t *const *flags, int32_t nflags, int64_t value,
                   const int64_t *value_dev, int64_t add, void *stream);
int ps_peer_wait(const int64_t *flags, int32_t nflags, int64_t value, const int64_t *value_dev,
                 int64_t add, int32_t *error, int64_t timeout_ns, void *stream);
int ps_peer_status(const int32_t *error);
size_t ps_ipc_handle_bytes(void);
int ps_ipc_export(const void *ptr, uint8_t *handle, int64_t *offset);
int ps_ipc_open(const uint8_t *handle, int64_t offset, void **ptr);

/* Device-resident per-stream frame counters for CUDA-graph replay (no host
 * scalar is baked into a captured frame).  state = int64[3]
 * {seq, frame_count, key}; one launch advances seq and frame_count by one and
 * sets key = (frame_count % gop_length == 0), the codec's key-frame rule
 * (codec.py:348).  Pass &state[0] as current_seq_dev and (int32_t *)&state[2]
 * as key_dev. */
int ps_frame_advance(int64_t *state, int64_t gop_length, void *stream);

/* Probe index buffer (the server module is absent from the
 * reference): uvarint(count), then per (slot, probe) entry sorted by slot
 * uvarint(slot - prev_slot) and uvarint(zigzag(probe - prev_probe)), prev
 * starting at (0, 0).  `out` holds >= 1 + 20 * max_entries bytes; the length
 * goes to the device scalar *out_len. */
size_t ps_index_workspace_bytes(int64_t max_entries);
int ps_encode_index(const int64_t *entries, const int64_t *entry_count, int64_t max_entries,
                    uint8_t *out, int64_t *out_len, void *workspace, size_t workspace_bytes,
                    void *stream);

/* Guard-band reconstruct over a whole atlas (packing.py:180-196 applied to
 * every probe block): rewrites each block's border from its core. */
int ps_reconstruct_guard_bands(int kind, void *atlas, int64_t probe_count,
                               int64_t probes_per_row, void *stream);

/* ---------------------------------------------------------------------------
 * Stages (1)+(2): probe ray tracing and DDGI blend (new API, no reference
 * implementation).
 * ------------------------------------------------------------------------- */

/* BVH: built on the host (binned SAH), uploaded by the shim. */
typedef struct ps_bvh_sizes {
    int64_t node_count;  /* nodes (size per layout, see ps_bvh_build_wide)   */
    int64_t tri_count;   /* triangles                                         */
    int64_t tri_slots;   /* 48-byte triangle records incl. leaf terminators   */
    int64_t max_depth;   /* deepest inner-node path (traversal stack bound)   */
} ps_bvh_sizes;

/* Build a BVH2 over `tri_count` triangles given as float64 vertices
 * (tri_count, 3, 3).  Writes host arrays: nodes (node_count * 16 floats),
 * tris (tri_slots * 12 floats).  Two-call protocol: pass NULL outputs to
 * query sizes. */
int ps_bvh_build(const double *vertices, int64_t tri_count, int leaf_size,
                 ps_bvh_sizes *sizes, float *nodes_out, float *tris_out);

/* Same with a node layout chosen by `width`:
 *   2  BVH2, 16-float nodes;
 *   4  BVH4, 32-float nodes: child boxes as lo.x[4] hi.x[4] lo.y[4] hi.y[4]
 *      lo.z[4] hi.z[4], child refs[4], pad[4]; unused slots have child
 *      0x7fffffff and the inverted box lo = +inf, hi = -inf;
 *   5  BVH4 with fp16 child boxes (16-float / 64-byte nodes: the same planes
 *      as halves, rounded outward, then child refs[4]) -- the default;
 *   3  BVH4 with fp16 boxes relative to an fp16 node origin and compact child
 *      references (64-byte nodes; measured slower, kept for comparison);
 *   8  BVH8 with 8-bit quantised boxes (24-float / 96-byte nodes; measured
 *      slower, kept for comparison).
 * Layouts 3 and 8 are documented in csrc/ps_bvh.cpp (emit_bvh4r / emit_bvh8).
 *
 * BVH frame (ABI 10): the builder uses the vertices as given.  The traversal
 * entry points (ps_trace_blend's `nodes`, ps_pvs) read a 64-byte header
 * placed immediately BEFORE node 0: its first three floats are the origin
 * of the frame the BVH was built in (the builder was given vertices minus
 * that origin; zeros for a world-frame BVH).  Rays are moved into that frame
 * for the traversal only.  scene.py builds around the scene's centre, which
 * halves the fp16 boxes' outward rounding. */
int ps_bvh_build_wide(const double *vertices, int64_t tri_count, int leaf_size, int width,
                      ps_bvh_sizes *sizes, float *nodes_out, float *tris_out);

/* Trace parameters (device pointers inside). */
typedef struct ps_trace_params {
    /* probe grid (volume.py:68-144) */
    int32_t nx, ny, nz;
    int32_t probe_begin;     /* first probe id handled (slab sharding)   */
    int32_t probe_end;       /* one past the last probe id handled       */
    double origin[3];
    double spacing[3];
    /* rays: directions for this frame (rays_per_probe, 4) float, shared by
     * every probe (one random rotation per frame) */
    const float *ray_dirs;
    int32_t rays_per_probe;
    /* scene */
    const float *nodes;      /* BVH node 0 (ps_bvh_build_wide layout), preceded
                              * by the 64-byte frame header (origin x, y, z) */
    int32_t bvh_width;       /* 2 or 4 */
    const float *tris;       /* triangle records */
    const float *materials;  /* per original triangle, 12 floats: albedo rgb _, emission
                              * rgb _, unit face normal xyz _ (normal in double, rounded) */
    int32_t light_count;
    const float *lights;     /* per light: position xyz, intensity rgb (6 floats) */
    float sky[3];
    float max_distance;
    float normal_bias;
    /* direct-light visibility at probe-ray hits:
     *   PS_SHADOW_NONE  unshadowed
     *   PS_SHADOW_RAYS  one any-hit shadow ray per light per hit
     *   PS_SHADOW_MAP   per-light cube distance maps traced from the light
     *                   each frame (the paper's server renders shadow maps,
     *                   PAPER.md:370), one lookup per light per hit */
    int32_t shadow_mode;
    int32_t shadow_map_size; /* cube face side S (PS_SHADOW_MAP)              */
    float *shadow_maps;      /* light_count * 6 * S * S distances (scratch)   */
    float shadow_bias;       /* relative slack of the map depth compare       */
    /* map texels [shadow_texel_begin, shadow_texel_end) of the flattened
     * (light, face, j, i) maps are traced (end 0 = all): ranks of a sharded
     * frame each trace a slice and all-gather the maps */
    int64_t shadow_texel_begin, shadow_texel_end;
    /* passes to run: bit 0 shadow maps, bit 1 probe rays, bit 2 blend; 0 = all */
    int32_t passes;
    /* blend */
    const float *w_color;    /* (rays, 64) cosine weights, transposed       */
    const float *w_depth;    /* (rays, 256) cosine^sharpness weights        */
    const float *inv_wsum;   /* (64 + 256) reciprocal weight sums            */
    /* optional tensor-core operand image of the weights written by
     * ps_blend_weights ((rays/8) * 6144 floats); non-NULL with rays % 8 == 0
     * selects the tcgen05 blend, NULL the CUDA-core blend */
    const float *w_image;
    float hysteresis;        /* 0 on the first frame                        */
    float irradiance_scale;  /* colour unorm = irradiance / scale            */
    /* state (float, persistent across frames), indexed by p - probe_begin */
    float *irradiance;       /* (probes, 64, 3)  */
    float *moments;          /* (probes, 256, 2) */
    /* outputs: atlases with guard bands (volume.py:147) */
    uint32_t *color_atlas;
    uint16_t *vis_atlas;
    int32_t probes_per_row_color;
    int32_t probes_per_row_vis;
    /* per-ray records written by the trace pass and read by the blend pass:
     * ((probe_end - probe_begin) * rays) float4 {radiance rgb, depth} */
    float *records;
    /* scratch: one uint32 work counter (dynamic ray-chunk scheduling) */
    uint32_t *work_counter;
    /* SMs the persistent trace grid leaves free for concurrent streams (the
     * previous frame's streaming stages) */
    int32_t reserve_sms;
    /* optional per-ray debug record ((probe_end - probe_begin) * rays, 8
     * floats: radiance rgb, depth, hit t (inf = miss), prim id (int bits,
     * -1 = miss), shadow mask (int bits, bit l = light l visible), 0);
     * NULL = off */
    float *ray_records;
    /* sharded shadow maps: when non-NULL the shadow pass stores each map texel
     * it traces into all shadow_ndst buffers (peers' maps mapped with CUDA
     * IPC, this rank's included) instead of shadow_maps */
    float *const *shadow_dst;
    int32_t shadow_ndst;
} ps_trace_params;

/* Per-frame weights: from ray_dirs and the texel directions
 * (texdir: 64*4 colour then 256*4 depth floats), writes w_color, w_depth,
 * inv_wsum, and (w_image != NULL, rays % 8 == 0) the tensor-core operand
 * image of ps_blend_weight_image_floats(rays) floats. */
int ps_blend_weights(const float *ray_dirs, int32_t rays_per_probe, const float *texdir,
                     float sharpness, float *w_color, float *w_depth, float *inv_wsum,
                     float *w_image, void *stream);
size_t ps_blend_weight_image_floats(int32_t rays_per_probe);

int ps_trace_blend(const ps_trace_params *params, void *stream);

/* Tuning only: traversal statistics gathered by the PS_TRACE_VARIANT=90
 * kernel, {inner-node visits, leaf visits, triangle tests, rays}; reset on
 * read. */
int ps_trace_stats(unsigned long long *out);

#ifdef __cplusplus
}
#endif

#endif /* PROBESTREAM_H */

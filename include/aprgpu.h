/* include/aprgpu.h -- C-ABI of the B200-native APR convolution path.
 *
 * This is the drop-in boundary for the reference's hot path (aprkit,
 * /root/reference/proj/include/aprkit).  Every entry point names the reference
 * interface it replaces.  Plain pointers, sizes and status codes only: no C++
 * types, no exceptions, no torch types cross this boundary.  The C++ shim a
 * maintainer adds on the reference side (include/aprkit_gpu.hpp) maps the
 * status codes back onto aprkit's exception taxonomy (errors.hpp:9-41).
 *
 * Conventions
 *  - Every function returns an aprgpu_status.  On failure the thread-local
 *    message is available from aprgpu_last_error().
 *  - Buffers flagged APRGPU_HOST are host memory (the call stages them through
 *    device memory and is synchronous); APRGPU_DEVICE buffers are device
 *    pointers on the APR's GPU and the call is stream-ordered on `stream`
 *    (a cudaStream_t; NULL = the context's own stream).
 *  - Thread-safe per context; one context per GPU.
 */
#ifndef APRGPU_H
#define APRGPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    APRGPU_OK = 0,
    APRGPU_ERR_RANGE = 1,      /* aprkit::RangeError      (errors.hpp:9-13)  */
    APRGPU_ERR_CAPABILITY = 2, /* aprkit::CapabilityError (errors.hpp:21-25) */
    APRGPU_ERR_INTEGRITY = 3,  /* aprkit::IntegrityError  (errors.hpp:15-19) */
    APRGPU_ERR_CUDA = 4,
    APRGPU_ERR_NCCL = 5,
    APRGPU_ERR_OOM = 6,
    APRGPU_ERR_INVALID = 7,    /* bad argument (null pointer, unknown enum, ...) */
    APRGPU_ERR_IO = 8,         /* aprkit::IoError            (errors.hpp:26-30) */
    APRGPU_ERR_BAD_FORMAT = 9, /* aprkit::BadFormatError     (errors.hpp:32-36) */
    APRGPU_ERR_TRUNCATED = 10  /* aprkit::TruncatedFileError (errors.hpp:38-41) */
} aprgpu_status;

enum { APRGPU_HOST = 0, APRGPU_DEVICE = 1 };
/* PadMode (reconstruct.hpp:13) */
enum { APRGPU_PAD_ZERO = 0, APRGPU_PAD_REFLECT = 1 };
/* Accumulation: EXACT = fp64 in the reference's (az,ax,ay) order, bit-identical
 * to convolve_apr; FAST = fp32 FMA in the same order (tolerance 1e-5 rel with
 * scale max(|e|,|g|,1) for non-negative stencils, acceptance.cpp:271-276). */
enum { APRGPU_ACCUM_EXACT = 0, APRGPU_ACCUM_FAST = 1 };
/* PyramidMode (stencil.hpp:162) */
enum { APRGPU_PYR_RESTRICTED = 0, APRGPU_PYR_RESCALED = 1, APRGPU_PYR_UNIFORM = 2, APRGPU_PYR_EXPLICIT = 3 };
/* which access structure */
enum { APRGPU_LEAF = 0, APRGPU_TREE = 1 };

#define APRGPU_MAX_LEVELS 20
#define APRGPU_MAX_EXTENT 13 /* kMaxStencilExtent, convolve.hpp:18 */

typedef struct aprgpu_ctx aprgpu_ctx;
typedef struct aprgpu_apr aprgpu_apr;
typedef struct aprgpu_pyramid aprgpu_pyramid;

/* Host view of aprkit::LinearAccess (linear_access.hpp:52-96): per-level dims
 * indexed by absolute level (l_max+1 entries), u16 y indices, u64 cumulative
 * row ends (one per (l,z,x) row), u64 level row offsets. */
typedef struct {
    int32_t l_min, l_max;
    const int32_t* z_dim;
    const int32_t* x_dim;
    const int32_t* y_dim;
    const uint16_t* y_idx;
    uint64_t n_particles;
    const uint64_t* xz_end;
    uint64_t n_rows;
    const uint64_t* level_offset;
} aprgpu_access_desc;

typedef struct {
    int32_t l_min, l_max;
    uint64_t n_particles, n_rows;
} aprgpu_access_info;

/* Page-locked host memory for callers' copy buffers (cudaHostAlloc,
 * portable): host-pointer calls copy such buffers directly instead of through
 * the context's staging -- per array, so pageable inputs with a page-locked
 * output (or the reverse) stage only the pageable side (new, no reference
 * counterpart). */
int aprgpu_host_alloc(uint64_t bytes, void** out);
int aprgpu_host_free(void* p);

/* ---- context ------------------------------------------------------------- */
int aprgpu_init(int device, aprgpu_ctx** out);
int aprgpu_ctx_free(aprgpu_ctx* ctx);
int aprgpu_ctx_stream(aprgpu_ctx* ctx, void** stream_out);
const char* aprgpu_last_error(void);
int aprgpu_version(void);

/* ---- structure ----------------------------------------------------------- */
/* Uploads the leaf access (aprkit::APR::access, apr.hpp:36) into the device
 * layout and builds everything the convolution needs (row-begin u32 prefix,
 * per-level non-empty row lists).  tree may be NULL: the interior-node
 * structure is then built on the GPU (replaces init_tree_structure,
 * tree.hpp:26-82, bit-exact); otherwise it is uploaded and its parent links are
 * verified (IntegrityError semantics of synchronized_parent_pass, tree.hpp:98). */
int aprgpu_upload_access(aprgpu_ctx* ctx, const aprgpu_access_desc* leaf, const aprgpu_access_desc* tree,
                         const int32_t source_dims[3], aprgpu_apr** out);
int aprgpu_apr_free(aprgpu_apr* apr);
int aprgpu_apr_dims(const aprgpu_apr* apr, int32_t dims_out[3]);
int aprgpu_access_get_info(const aprgpu_apr* apr, int which, aprgpu_access_info* out);
/* Resident gather maps of the tile kernel: *built = tile records held over all
 * (stencil extent, pad mode, level) maps, *n_tiles = the APR's output tiles.  A
 * z-slab's convolutions build records only for the tiles they compute. */
int aprgpu_apr_map_tiles(const aprgpu_apr* apr, uint64_t* built, uint64_t* n_tiles);
/* Restricts the APR's per-tile convolution state (tile probe, source runs,
 * staged-source lists, gather maps) to the tiles meeting finest-level planes
 * [z_lo, z_hi) at levels >= cut_level (levels below whole): a z-slab rank
 * builds and holds ~1/N of it.  Must precede the first convolution; a later
 * convolution outside the slab fails with APRGPU_ERR_CAPABILITY. */
int aprgpu_apr_restrict(aprgpu_apr* apr, int cut_level, int32_t z_lo, int32_t z_hi);
/* Diagnostics: copies the resident gather-map records of one level (stencil
 * half-width 1 or 2, pad mode) to host memory out (cap_words u32), record t
 * starting at word offsets[t] (offsets: *n_tiles + 1 entries); *n_words = the words copied, *first_tile
 * / *n_tiles = the level-local tile range covered (0 tiles: no map built yet).
 * out and offsets may be NULL to query sizes first. */
int aprgpu_map_records(const aprgpu_apr* apr, int half_width, int pad, int level, uint32_t* out,
                       uint64_t cap_words, uint32_t* offsets, uint64_t* n_words, uint64_t* first_tile,
                       uint64_t* n_tiles);
/* Downloads an access structure back into the reference layout (bit-exact
 * round trip).  Arrays sized by aprgpu_access_get_info: y_idx[n_particles],
 * xz_end[n_rows], level_offset/z_dim/x_dim/y_dim[l_max+1]. */
int aprgpu_download_access(const aprgpu_apr* apr, int which, uint16_t* y_idx, uint64_t* xz_end,
                           uint64_t* level_offset, int32_t* z_dim, int32_t* x_dim, int32_t* y_dim);
/* nonempty_row_index (convolve.hpp:32-44) for one level: writes up to cap rows
 * (z, x, y_min, y_max) and returns the row count in *count. */
int aprgpu_row_index(const aprgpu_apr* apr, int level, int32_t* z, int32_t* x, uint16_t* y_min,
                     uint16_t* y_max, uint64_t cap, uint64_t* count);

/* The per-call index step of the paper's GPU protocol ("row
 * index + tree fill + convolution"): nonempty_row_index (convolve.hpp:32-44)
 * for every level plus the occupied-tile lists derived from it, recomputed on
 * the device into APR scratch, stream-ordered (no host synchronisation).  The
 * convolution keeps using the identical lists built at upload; this entry
 * point exists so a protocol that counts the index step can time it. */
int aprgpu_rebuild_index(aprgpu_apr* apr, void* stream);

/* ---- tree ----------------------------------------------------------------- */
/* fill_tree (tree.hpp:110-150): leaf[n_particles] -> tree[n_tree]; fp64
 * accumulation in the reference's per-parent order, bit-exact. */
int aprgpu_fill_tree(aprgpu_apr* apr, const float* leaf, float* tree, int ptr_kind, void* stream);

/* ---- dense pixel convolution (convolve.hpp:48-98) --------------------------- */
/* convolve_pixels: out = w * in over an nz x nx x ny volume ((z, x, y), y fastest),
 * true-convolution convention, reflect / zero padding, taps in the reference's
 * order skipping zero weights; EXACT accumulation is bit-identical.  w[kz*kx*ky]
 * is always a host array.  CAPABILITY: an extent above 13; RANGE: even extents. */
int aprgpu_convolve_pixels(aprgpu_ctx* ctx, const float* in, int nz, int nx, int ny, const float* w, int kz, int kx,
                           int ky, int pad_mode, int accum, float* out, int ptr_kind, void* stream);

/* ---- .apr container (io.hpp:102-183, docs/FORMATS.md) ---------------------- */
/* BuildParams (apr.hpp:16-33) as stored in an .apr file: sigma_mode 0 constant /
 * 1 local range; gradient_mode 0 central difference / 1 Sobel. */
typedef struct {
    double rel_error;
    int sigma_mode;
    double sigma_value;
    int sigma_window;
    double sigma_floor;
    int gradient_mode;
    int smoothing_passes;
} aprgpu_build_params;

/* load_apr / read_apr (io.hpp:131-183): the file straight into a device handle
 * -- leaf and interior structure as stored, leaf values on the device
 * (aprgpu_apr_values), build parameters (aprgpu_apr_params) -- after the
 * reader's checks (same order and messages) and validate on the device.
 * Errors: IO (cannot open), BAD_FORMAT (malformed, or validate's violation
 * as "invalid APR structure: ..."), TRUNCATED (early end of file). */
int aprgpu_load_apr(aprgpu_ctx* ctx, const char* path, aprgpu_apr** out);
/* save_apr / write_apr (io.hpp:106-126, 171-176): values[n_particles] (host or
 * device) with the handle's structure and parameters; byte-identical to the
 * reference's writer.  Handles not loaded from a file carry BuildParams'
 * defaults, or build_apr's (E, constant sigma = intensity range). */
int aprgpu_save_apr(aprgpu_apr* apr, const char* path, const float* values, int ptr_kind);
int aprgpu_apr_params(const aprgpu_apr* apr, aprgpu_build_params* out);

/* validate (apr.hpp:61-134) of a leaf access and its image dims, on the device
 * in O(particles + rows) instead of the reference's O(pixels) cover map: *ok = 1,
 * or 0 with the reference's message for the first violation it reports copied
 * to msg (msg_cap bytes, NUL-terminated; msg may be NULL).  Violations are
 * results, not errors; errors are the usual status codes. */
int aprgpu_validate_access(aprgpu_ctx* ctx, const aprgpu_access_desc* leaf, const int32_t source_dims[3], int* ok,
                           char* msg, size_t msg_cap);

/* ---- dense reconstruction (reconstruct.hpp:73-129) ------------------------- */
/* Patch window of reconstruct_patch (PatchSpec, reconstruct.hpp:28-35): level-l
 * cells z in [z_begin, z_end), x in [x_begin, x_end), the full y span, pad cells
 * per side filled by pad_mode (APRGPU_PAD_ZERO / APRGPU_PAD_REFLECT). */
typedef struct {
    int level, z_begin, z_end, x_begin, x_end, pad, pad_mode;
} aprgpu_patch_spec;

/* reconstruct_level (reconstruct.hpp:73-84): out[z_dim(l) * x_dim(l) * y_dim(l)],
 * (z, x, y) at (z * x_dim + x) * y_dim + y.  Every cell takes its covering leaf's
 * value (fill_level_row, :41-69), or with tree_values its level-l interior
 * node's; tree_values NULL writes no interior nodes (reconstruct_full is
 * level l_max with NULL).  RANGE: level outside [l_min, l_max]. */
int aprgpu_reconstruct_level(aprgpu_apr* apr, const float* values, const float* tree_values, int level, float* out,
                             int ptr_kind, void* stream);
/* reconstruct_patch (reconstruct.hpp:94-129): out[(z_end - z_begin + 2 pad) *
 * (x_end - x_begin + 2 pad) * (y_dim(l) + 2 pad)].  RANGE: spec outside the grid. */
int aprgpu_reconstruct_patch(aprgpu_apr* apr, const float* values, const float* tree_values,
                             const aprgpu_patch_spec* spec, float* out, int ptr_kind, void* stream);

/* ---- stencils (host) ------------------------------------------------------ */
/* restrict_stencil (stencil.hpp:127-160).  out_k3 gets the restricted extents;
 * out (may be NULL to query) gets the weights, bit-identical to the reference
 * wherever the reference's O(8^delta k^3) loop is tractable. */
int aprgpu_restrict_stencil(const float* w, int kz, int kx, int ky, int delta, int32_t out_k3[3], float* out);
/* gaussian_stencil (stencil.hpp:59-79), box_stencil (:52), sobel_stencil (:83) */
int aprgpu_gaussian_stencil(double sigma, int size, int32_t* k_out, float* out);
int aprgpu_box_stencil(int k, float* out);
int aprgpu_sobel_stencil(int axis, float* out);

/* make_pyramid (stencil.hpp:176-191) / explicit_pyramid (:193-202), held on
 * the device for the convolution.  For explicit pyramids w holds the stencils
 * level by level, k3 their extents (3 ints per level). */
int aprgpu_pyramid_create(aprgpu_ctx* ctx, const float* w, int kz, int kx, int ky, int l_min, int l_max,
                          int mode, aprgpu_pyramid** out);
int aprgpu_pyramid_create_explicit(aprgpu_ctx* ctx, const float* w, const int32_t* k3, int l_min, int l_max,
                                   aprgpu_pyramid** out);
int aprgpu_pyramid_free(aprgpu_pyramid* p);
/* StencilPyramid::at (stencil.hpp:170-173): extents and (optionally) weights */
int aprgpu_pyramid_level(const aprgpu_pyramid* p, int level, int32_t k3[3], float* w);

/* ---- convolution ---------------------------------------------------------- */
/* convolve_apr (convolve.hpp:220-303): out[n_particles] from values[n_particles]
 * and tree_values[n_tree].  accum: APRGPU_ACCUM_EXACT (bit-identical to the
 * reference) or APRGPU_ACCUM_FAST.  Errors: RANGE if the pyramid does not cover
 * the APR levels (:224-225), CAPABILITY if an extent exceeds 13 (:226-230). */
int aprgpu_convolve(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                    int pad_mode, int accum, float* out, int ptr_kind, void* stream);

/* rl_apr (deconv.hpp:75-107): iterations of fill_tree -> conv(w) -> ratio ->
 * fill_tree -> conv(flip w) -> multiply, all on the device.  psf is normalised
 * like normalized_psf (:26-34).  epsilon <= 0 selects 1e-6 x mean(observed)
 * (rl_epsilon, :36-38).  out[n_particles]. */
int aprgpu_rl(aprgpu_apr* apr, const float* observed, const float* psf, int kz, int kx, int ky, int iterations,
              double epsilon, int accum, float* out, int ptr_kind, void* stream);

/* ---- z-slab decomposition (multi-GPU) ----------------------
 * Every rank holds the whole structure; a slab is the finest-level pixel
 * planes [z_lo, z_hi) (z_lo, z_hi multiples of 2^(l_max - lc)).  Levels >= lc
 * are partitioned (a cell fits in a slab), levels < lc are replicated.  All
 * buffers are device pointers in the global particle / node numbering.
 *
 * fp64 tree sums of interior levels [lt_lo, lt_hi], parent rows in the slab
 * only (z_hi < 0: all rows); the scratch holds n_tree doubles each and is what
 * ranks exchange at the cut level. */
int aprgpu_fill_tree_sums(aprgpu_apr* apr, const float* leaf, int lt_lo, int lt_hi, int z_lo, int z_hi,
                          void* stream);
int aprgpu_tree_scratch(aprgpu_apr* apr, double** vsum, double** wsum);
/* tree[i] = float(vsum[i] / wsum[i]) (0 when wsum is 0), tree.hpp:146-148 */
int aprgpu_fill_tree_finalize(aprgpu_apr* apr, float* tree, void* stream);
/* convolve_apr computing the outputs of levels >= lc in the slab's rows and of
 * every level < lc; other outputs are left untouched. */
int aprgpu_convolve_slab(aprgpu_apr* apr, const float* values, const float* tree_values, const aprgpu_pyramid* pyr,
                         int pad_mode, int accum, int lc, int z_lo, int z_hi, float* out, void* stream);
/* The same over a band of a slab, the replicated levels < lc computed only when
 * `replicated` is nonzero: how a rank convolves its interior (planes at least
 * halo * 2^(l_max - lc) from a cut) while the halo exchange is in flight, then
 * its boundary bands once the halos have landed. */
int aprgpu_convolve_slab_band(aprgpu_apr* apr, const float* values, const float* tree_values,
                              const aprgpu_pyramid* pyr, int pad_mode, int accum, int lc, int z_lo, int z_hi,
                              int replicated, float* out, void* stream);

/* ---- multi-GPU z-slabs in one process (csrc/multi.cu) -------
 * The volume cut into n_slabs z-slabs, slab s on device devices[s] (entries
 * may repeat: several slabs on one GPU); every device holds the structure,
 * levels >= the cut level are partitioned, coarser ones replicated, and the
 * halo -- `halo` rows of every partitioned level, at least the stencils'
 * half-width -- is copied peer to peer (NVLink / NVSwitch) while each slab's
 * interior already convolves.  tree may be NULL (built on the devices).
 * convolve_apr (convolve.hpp:220-303) over the slabs: HOST values[n_particles]
 * and tree_values[n_tree] in, out[n_particles] out; the pyramid is explicit
 * (w: level-by-level weights, k3: 3 extents per level, levels l_min..l_max).
 * Bit-identical to aprgpu_convolve in EXACT mode.  RANGE: the volume is too
 * thin for the slab count, or a stencil half-width exceeds the halo. */
typedef struct aprgpu_multi aprgpu_multi;
int aprgpu_multi_create(const int* devices, int n_slabs, const aprgpu_access_desc* leaf,
                        const aprgpu_access_desc* tree, const int32_t source_dims[3], int halo, aprgpu_multi** out);
int aprgpu_multi_free(aprgpu_multi* m);
/* n_slabs, the cut level and each slab's finest-level planes [z_bounds[2s], z_bounds[2s+1]) */
int aprgpu_multi_info(const aprgpu_multi* m, int* n_slabs, int* cut_level, int32_t* z_bounds);
int aprgpu_multi_convolve(aprgpu_multi* m, const float* values, const float* tree_values, const float* w,
                          const int32_t* k3, int l_min, int l_max, int pad_mode, int accum, float* out);

/* rl_apr resumed from a running estimate (estimate_in[n_particles]; NULL =
 * start from the clamped observation, i.e. aprgpu_rl).  The reference's state
 * between iterations is exactly (u, epsilon, estimate), so running k iterations
 * and resuming for m more is bit-identical to k + m iterations: this is how the
 * C++ drop-in serves rl_apr's observer (deconv.hpp:103-104). */
int aprgpu_rl_resume(aprgpu_apr* apr, const float* observed, const float* estimate_in, const float* psf, int kz,
                     int kx, int ky, int iterations, double epsilon, int accum, float* out, int ptr_kind,
                     void* stream);
/* rl_apr's observation sum (deconv.hpp:90-91: `double mean = 0; for (float v :
 * u) mean += v;`) of n non-negative values, bit-identical to that sequential
 * loop, computed on the device (the parallel replay rl_apr falls back to when
 * its partial sums are not provably exact).  RANGE for a negative or non-finite
 * value.  Synchronises the stream. */
int aprgpu_sequential_sum(aprgpu_ctx* ctx, const float* values, uint64_t n, int ptr_kind, double* out, void* stream);

/* ---- inputs: synthetic volumes and APR construction (input side of the path) */
/* generate_spheres (synthetic.hpp:74-111, no noise) into out[nz*nx*ny] (z,x,y
 * order, y fastest), on the device; bit-identical to the reference volume. */
int aprgpu_generate_spheres(aprgpu_ctx* ctx, int nz, int nx, int ny, int count, double min_radius,
                            double max_radius, double background, double min_intensity, double max_intensity,
                            double blur_sigma, uint64_t seed, float* out, int ptr_kind);
/* build_apr (build.hpp:290-312) with SigmaPolicy::constant(intensity_range(v)),
 * central-difference gradient and no smoothing, on the device: pixels ->
 * leaf access + interior access + sampled particle values (aprgpu_apr_values). */
int aprgpu_build_apr(aprgpu_ctx* ctx, const float* volume, int nz, int nx, int ny, double rel_error, int ptr_kind,
                     aprgpu_apr** out);
/* build_apr (build.hpp:290-312) with any BuildParams (apr.hpp:16-33), on the
 * device: gradient_magnitude central differences or Sobel (:42-75),
 * smoothing_passes 3^3 box passes (:22-38, :298), local_scale constant or
 * local range with its box smoothing and floor (:80-108), level_function
 * (:113-129) with the constant-sigma safety level, then solve_levels,
 * init_tree_structure and sample_particles -- structure and values
 * bit-identical to the reference (a reference compiled with
 * -ffp-contract=off).  aprgpu_build_apr is this with
 * SigmaPolicy::constant(intensity_range(volume)) and the other defaults. */
int aprgpu_build_apr_params(aprgpu_ctx* ctx, const float* volume, int nz, int nx, int ny,
                            const aprgpu_build_params* params, int ptr_kind, aprgpu_apr** out);
/* The C4 tiler: a power-of-two cube APR tiled (tz, tx, ty) times into a new
 * APR built directly in the device layout (structure + interior structure),
 * and the matching tiling of particle values (device pointers; big_values
 * holds n_particles of the tiled APR). */
int aprgpu_tile_apr(aprgpu_apr* src, int tz, int tx, int ty, aprgpu_apr** out);
int aprgpu_tile_values(aprgpu_apr* src, aprgpu_apr* big, int tz, int tx, int ty, const float* src_values,
                       float* big_values);

/* Copies the particle values sampled by aprgpu_build_apr (sample_particles,
 * build.hpp:252-284) or read by aprgpu_load_apr into out[n_particles]. */
int aprgpu_apr_values(const aprgpu_apr* apr, float* out, int ptr_kind);

/* Number of kernel launches this context issued since creation (bench.py's
 * gpu_launches evidence). */
int aprgpu_launch_count(aprgpu_ctx* ctx, uint64_t* out);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif

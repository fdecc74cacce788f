/* oracle/aprk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (aprkit, /root/reference/proj) algorithms
 * on the APR convolution hot path.  Used exclusively as the checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg; the product never
 * links or calls it.  Every function cites the reference file:line it follows.
 *
 * Parity pinning: tests/test_oracle.py checks every function here bit-for-bit
 * against (a) the committed golden vectors in tests/golden/ (produced by the
 * real reference through oracle/_ref, script tests/golden/make_golden.py) and
 * (b) the live reference library oracle/_ref/libaprref.so when present.
 */
#ifndef APRK_ORACLE_H
#define APRK_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat view of aprkit::LinearAccess (linear_access.hpp:52-96). */
typedef struct {
    int l_min, l_max;
    const int* z_dim; /* l_max+1 */
    const int* x_dim;
    const int* y_dim;
    const uint16_t* y_idx;
    uint64_t n_particles;
    const uint64_t* xz_end;
    uint64_t n_rows;
    const uint64_t* level_offset; /* l_max+1 */
} orc_access;

/* validate (apr.hpp:61-134): 1 if ok, else 0 with the reference's message in msg */
int orc_validate(const orc_access* a, const int dims[3], char* msg, size_t cap);

/* reflect_index (reconstruct.hpp:17-25) */
int orc_reflect_index(int i, int n);

/* get_row (linear_access.hpp:70-80); returns 0 or -1 (RangeError) */
int orc_get_row(const orc_access* a, int l, int z, int x, uint64_t* begin, uint64_t* end);

/* init_tree_structure (tree.hpp:26-82).  Two-phase: orc_tree_structure_count
 * computes the per-row counts (n_rows_out entries, rows of levels
 * t_l_min..t_l_max) and returns the tree level range; orc_tree_structure_fill
 * writes y_idx.  Simpler: orc_init_tree_structure allocates with malloc. */
typedef struct {
    int l_min, l_max;
    int* z_dim; int* x_dim; int* y_dim;
    uint16_t* y_idx; uint64_t n_particles;
    uint64_t* xz_end; uint64_t n_rows;
    uint64_t* level_offset;
} orc_owned_access;
int orc_init_tree_structure(const orc_access* leaf, const int dims[3], orc_owned_access* out);
void orc_free_access(orc_owned_access* a);

/* fill_tree (tree.hpp:110-150).  Returns 0, or -3 on a missing parent
 * (IntegrityError, tree.hpp:98-100). */
int orc_fill_tree(const orc_access* leaf, const orc_access* tree, const int dims[3],
                  const float* leaf_values, float* tree_out);

/* nonempty_row_index (convolve.hpp:32-44) for one level; returns the count and
 * writes up to cap entries when the arrays are non-null. */
int64_t orc_nonempty_rows(const orc_access* a, int level, int* z, int* x, uint16_t* ymin,
                          uint16_t* ymax, int64_t cap);

/* fill_level_row (reconstruct.hpp:41-69) */
void orc_fill_level_row(const orc_access* leaf, const float* values, const orc_access* tree,
                        const float* tree_values, int l, int z, int x, float* dst, int y_begin,
                        int y_end);

/* reconstruct_level (reconstruct.hpp:73-84): out is z_dim*x_dim*y_dim at l */
void orc_reconstruct_level(const orc_access* leaf, const float* values, const orc_access* tree,
                           const float* tree_values, int l, float* out);

/* reconstruct_patch (reconstruct.hpp:94-129): spec = level, z_begin, z_end,
 * x_begin, x_end, pad, pad_mode (0 Zero, 1 Reflect); out is (z_end - z_begin +
 * 2 pad) x (x_end - x_begin + 2 pad) x (y_dim + 2 pad).  tree_values may be NULL. */
void orc_reconstruct_patch(const orc_access* leaf, const float* values, const orc_access* tree,
                           const float* tree_values, const int spec[7], float* out);

/* convolve_pixels (convolve.hpp:48-98): out[nz*nx*ny]; pad 0 Zero, 1 Reflect */
void orc_convolve_pixels(const float* v, int nz, int nx, int ny, const float* w, int kz, int kx, int ky,
                         int pad, float* out);

/* restrict_stencil (stencil.hpp:127-160).  out_k3 receives the extents; out may
 * be NULL to query them. */
void orc_restrict_stencil(const float* w, int kz, int kx, int ky, int delta, int out_k3[3],
                          float* out);

/* Per-level stencil pyramid as consumed by orc_convolve: level l uses
 * k3[3*(l-l_min)..] and weights at w + off[l-l_min]. */
typedef struct {
    int l_min, l_max;
    const int* k3;
    const float* w;
    const uint64_t* off;
} orc_pyramid;

/* convolve_apr (convolve.hpp:220-303): exact restatement of the per-level
 * reconstruction + (az,ax,ay)-ordered fp64 accumulation of LevelSlab::apply
 * (convolve.hpp:154-169).  pad: 0 Zero, 1 Reflect.  Returns 0, -1 RangeError,
 * -2 CapabilityError. */
int orc_convolve(const orc_access* leaf, const orc_access* tree, const float* values,
                 const float* tree_values, const orc_pyramid* pyr, int pad, float* out);

/* rl_apr (deconv.hpp:75-107) with explicit pyramids for w and flip(w) (built
 * by the caller with orc_restrict_stencil).  eps as computed by rl_epsilon. */
int orc_rl_apr(const orc_access* leaf, const orc_access* tree, const int dims[3],
               const float* observed, const orc_pyramid* pyr_w, const orc_pyramid* pyr_wt,
               int iterations, double eps, float* out);

/* generate_spheres (synthetic.hpp:74-111, no noise) into v[nz*nx*ny] and
 * build_apr (build.hpp:290-312; constant sigma = intensity range, central
 * differences, no smoothing) -> leaf access (malloc'd; orc_free_access) and
 * sampled values (orc_free_values).  Multi-threaded over z planes, bit-identical
 * to the reference (build_oracle.c).  Return 0, or -1 on bad input / no memory. */
int orc_generate_spheres(int nz, int nx, int ny, int count, double min_r, double max_r, double background,
                         double min_i, double max_i, double blur, uint64_t seed, int threads, float* v);
int orc_build_apr(const float* v, int nz, int nx, int ny, double rel_error, int threads, orc_owned_access* out,
                  float** values_out);
void orc_free_values(float* v);

#ifdef __cplusplus
}
#endif
#endif

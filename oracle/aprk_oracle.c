/* oracle/aprk_oracle.c -- TEST INFRASTRUCTURE ONLY (see aprk_oracle.h).
 *
 * A deliberately plain, single-threaded C restatement of the reference
 * algorithms.  Performance is irrelevant here; faithfulness to the reference's
 * arithmetic (operation order, rounding points) is everything.
 */
#include "aprk_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_EXTENT 13 /* kMaxStencilExtent, convolve.hpp:18 */

int orc_reflect_index(int i, int n) { /* reconstruct.hpp:17-25 */
    while (i < 0 || i >= n) i = (i < 0) ? (-i - 1) : (2 * n - 1 - i);
    return i;
}

static int cell_size(int l_max, int l) { return 1 << (l_max - l); }                 /* linear_access.hpp:19 */
static int grid_dim(int n, int l_max, int l) { int s = cell_size(l_max, l); return (n + s - 1) / s; } /* :21-24 */
static int compute_l_max(int nz, int nx, int ny) {                                  /* :27-32 */
    int m = nz > nx ? nz : nx;
    if (ny > m) m = ny;
    int l = 0;
    while ((1 << l) < m) ++l;
    return l;
}

int orc_get_row(const orc_access* a, int l, int z, int x, uint64_t* begin, uint64_t* end) {
    /* linear_access.hpp:70-80: row r covers [xz_end[r-1], xz_end[r]), row 0 begins at 0 */
    if (l < a->l_min || l > a->l_max) return -1;
    if (z < 0 || z >= a->z_dim[l] || x < 0 || x >= a->x_dim[l]) return -1;
    uint64_t r = a->level_offset[l] + (uint64_t)z * (uint64_t)a->x_dim[l] + (uint64_t)x;
    *begin = r ? a->xz_end[r - 1] : 0;
    *end = a->xz_end[r];
    return 0;
}

/* validate (apr.hpp:61-134): the reference's checks in its order, with its
 * messages (into msg, cap bytes); the partition property by marking every pixel
 * (O(pixels): this is the checker, not the product).  Returns 1 if ok. */
int orc_validate(const orc_access* a, const int dims[3], char* msg, size_t cap) {
#define ORC_FAIL(...) do { if (msg && cap) snprintf(msg, cap, __VA_ARGS__); return 0; } while (0)
    if (msg && cap) msg[0] = 0;
    if (a->l_min > a->l_max) ORC_FAIL("l_min > l_max");
    uint64_t expect = 0;
    for (int l = a->l_min; l <= a->l_max; ++l) {
        if (a->level_offset[l] != expect) ORC_FAIL("level_offset mismatch at level %d", l);
        expect += (uint64_t)a->z_dim[l] * (uint64_t)a->x_dim[l];
    }
    if (a->n_rows != expect) ORC_FAIL("xz_end length does not match level grids");
    uint64_t prev = 0;
    for (uint64_t r = 0; r < a->n_rows; ++r) {
        if (a->xz_end[r] < prev) ORC_FAIL("xz_end decreases at row %llu", (unsigned long long)r);
        prev = a->xz_end[r];
    }
    if (a->n_rows && a->xz_end[a->n_rows - 1] != a->n_particles) ORC_FAIL("xz_end[last] != y_idx length");
    if (!a->n_rows && a->n_particles) ORC_FAIL("particles present but no rows");
    for (int l = a->l_min; l <= a->l_max; ++l)
        for (int z = 0; z < a->z_dim[l]; ++z)
            for (int x = 0; x < a->x_dim[l]; ++x) {
                uint64_t b, e;
                orc_get_row(a, l, z, x, &b, &e);
                int last = -1;
                for (uint64_t i = b; i < e; ++i) {
                    const int y = a->y_idx[i];
                    if (y <= last) ORC_FAIL("non-increasing y in row (%d, %d, %d)", l, z, x);
                    if (y >= a->y_dim[l]) ORC_FAIL("y index out of level grid in level %d", l);
                    last = y;
                }
            }
    const uint64_t n_pixels = (uint64_t)dims[0] * (uint64_t)dims[1] * (uint64_t)dims[2];
    if (n_pixels == 0) return 1;
    uint8_t* cover = (uint8_t*)calloc(n_pixels, 1);
    int dbl = 0, overflow = 0;
    for (int l = a->l_min; l <= a->l_max; ++l) {
        const int s = 1 << (a->l_max - l);  /* cell_size(geom_l_max = l_max, l) */
        for (int z = 0; z < a->z_dim[l]; ++z)
            for (int x = 0; x < a->x_dim[l]; ++x) {
                uint64_t b, e;
                orc_get_row(a, l, z, x, &b, &e);
                for (uint64_t i = b; i < e; ++i) {
                    const int64_t z0 = (int64_t)z * s, x0 = (int64_t)x * s, y0 = (int64_t)a->y_idx[i] * s;
                    if (z0 >= dims[0] || x0 >= dims[1] || y0 >= dims[2]) { overflow = 1; continue; }
                    const int64_t z1 = z0 + s < dims[0] ? z0 + s : dims[0];
                    const int64_t x1 = x0 + s < dims[1] ? x0 + s : dims[1];
                    const int64_t y1 = y0 + s < dims[2] ? y0 + s : dims[2];
                    for (int64_t zz = z0; zz < z1; ++zz)
                        for (int64_t xx = x0; xx < x1; ++xx)
                            for (int64_t yy = y0; yy < y1; ++yy) {
                                uint8_t* c = cover + ((uint64_t)zz * dims[1] + (uint64_t)xx) * dims[2] + (uint64_t)yy;
                                if (*c) dbl = 1;
                                *c = 1;
                            }
                }
            }
    }
    int ok = 1;
    if (overflow) { if (msg && cap) snprintf(msg, cap, "particle cell outside the image domain"); ok = 0; }
    else if (dbl) { if (msg && cap) snprintf(msg, cap, "double coverage: overlapping particle cells"); ok = 0; }
    else
        for (uint64_t i = 0; i < n_pixels; ++i)
            if (!cover[i]) {
                if (msg && cap) snprintf(msg, cap, "uncovered pixel at flat index %llu", (unsigned long long)i);
                ok = 0;
                break;
            }
    free(cover);
    return ok;
#undef ORC_FAIL
}

/* ---------------------------------------------------------------- tree ---- */

static int cmp_u16(const void* p, const void* q) {
    int a = *(const uint16_t*)p, b = *(const uint16_t*)q;
    return a - b;
}

int orc_init_tree_structure(const orc_access* leaf, const int dims[3], orc_owned_access* out) {
    /* tree.hpp:26-82.  Interior nodes on levels [max(l_min-1,0), l_max-1]; a
     * parent row is the sorted unique set of (child y)/2 over its 2x2 (z,x)
     * child rows, leaves and interior nodes alike, built finest first. */
    memset(out, 0, sizeof(*out));
    const int glm = leaf->l_max;
    const int tmax = leaf->l_max - 1;
    const int tmin = leaf->l_min - 1 > 0 ? leaf->l_min - 1 : 0;
    /* geometry of assemble_access (linear_access.hpp:110-119) */
    int geom = glm;
    int cl = compute_l_max(dims[0], dims[1], dims[2]);
    if (cl > geom) geom = cl;
    if (tmax < tmin) { /* tree.hpp:31-42: single-cell edge case */
        out->l_min = 0; out->l_max = 0;
        out->z_dim = calloc(1, sizeof(int)); out->x_dim = calloc(1, sizeof(int)); out->y_dim = calloc(1, sizeof(int));
        out->z_dim[0] = grid_dim(dims[0], glm, 0);
        out->x_dim[0] = grid_dim(dims[1], glm, 0);
        out->y_dim[0] = grid_dim(dims[2], glm, 0);
        out->level_offset = calloc(1, sizeof(uint64_t));
        out->n_rows = (uint64_t)out->z_dim[0] * out->x_dim[0];
        out->xz_end = calloc(out->n_rows ? out->n_rows : 1, sizeof(uint64_t));
        out->y_idx = malloc(1);
        return 0;
    }
    /* per-level row lists (vector of uint16 per row) */
    uint16_t*** rows = calloc((size_t)tmax + 1, sizeof(uint16_t**));
    uint32_t** lens = calloc((size_t)tmax + 1, sizeof(uint32_t*));
    for (int lt = tmax; lt >= tmin; --lt) {
        const int zd = grid_dim(dims[0], glm, lt), xd = grid_dim(dims[1], glm, lt);
        const int c = lt + 1;
        const int czd = grid_dim(dims[0], glm, c), cxd = grid_dim(dims[1], glm, c);
        rows[lt] = calloc((size_t)zd * xd, sizeof(uint16_t*));
        lens[lt] = calloc((size_t)zd * xd, sizeof(uint32_t));
        for (int z = 0; z < zd; ++z)
            for (int x = 0; x < xd; ++x) {
                size_t cap = 0, n = 0;
                uint16_t* ys = NULL;
                for (int cz = 2 * z; cz < 2 * z + 2 && cz < czd; ++cz)
                    for (int cx = 2 * x; cx < 2 * x + 2 && cx < cxd; ++cx) {
                        uint64_t b = 0, e = 0;
                        size_t add = 0;
                        const uint16_t* src = NULL;
                        const uint16_t* tsrc = NULL;
                        size_t tn = 0;
                        if (c >= leaf->l_min && c <= leaf->l_max) {
                            orc_get_row(leaf, c, cz, cx, &b, &e);
                            src = leaf->y_idx + b;
                            add += (size_t)(e - b);
                        }
                        if (c <= tmax) {
                            tsrc = rows[c][(size_t)cz * cxd + cx];
                            tn = lens[c][(size_t)cz * cxd + cx];
                            add += tn;
                        }
                        if (n + add > cap) {
                            cap = (n + add) * 2 + 8;
                            ys = realloc(ys, cap * sizeof(uint16_t));
                        }
                        for (uint64_t i = 0; src && i < e - b; ++i) ys[n++] = (uint16_t)(src[i] / 2);
                        for (size_t i = 0; i < tn; ++i) ys[n++] = (uint16_t)(tsrc[i] / 2);
                    }
                if (n) qsort(ys, n, sizeof(uint16_t), cmp_u16);
                size_t u = 0;
                for (size_t i = 0; i < n; ++i)
                    if (u == 0 || ys[u - 1] != ys[i]) ys[u++] = ys[i];
                rows[lt][(size_t)z * xd + x] = ys;
                lens[lt][(size_t)z * xd + x] = (uint32_t)u;
            }
    }
    /* assemble_access(tmin, tmax, dims, rows) (linear_access.hpp:101-130) */
    out->l_min = tmin;
    out->l_max = tmax;
    out->z_dim = calloc((size_t)tmax + 1, sizeof(int));
    out->x_dim = calloc((size_t)tmax + 1, sizeof(int));
    out->y_dim = calloc((size_t)tmax + 1, sizeof(int));
    out->level_offset = calloc((size_t)tmax + 1, sizeof(uint64_t));
    uint64_t nr = 0, np = 0;
    for (int lt = tmin; lt <= tmax; ++lt) {
        const int zd = grid_dim(dims[0], geom, lt), xd = grid_dim(dims[1], geom, lt);
        for (size_t r = 0; r < (size_t)zd * xd; ++r) np += lens[lt][r];
        nr += (uint64_t)zd * xd;
    }
    out->n_rows = nr;
    out->n_particles = np;
    out->xz_end = malloc((nr ? nr : 1) * sizeof(uint64_t));
    out->y_idx = malloc((np ? np : 1) * sizeof(uint16_t));
    uint64_t row = 0, p = 0;
    for (int lt = tmin; lt <= tmax; ++lt) {
        const int zd = grid_dim(dims[0], geom, lt), xd = grid_dim(dims[1], geom, lt);
        out->z_dim[lt] = zd;
        out->x_dim[lt] = xd;
        out->y_dim[lt] = grid_dim(dims[2], geom, lt);
        out->level_offset[lt] = row;
        for (size_t r = 0; r < (size_t)zd * xd; ++r, ++row) {
            memcpy(out->y_idx + p, rows[lt][r], lens[lt][r] * sizeof(uint16_t));
            p += lens[lt][r];
            out->xz_end[row] = p;
            free(rows[lt][r]);
        }
        free(rows[lt]);
        free(lens[lt]);
    }
    free(rows);
    free(lens);
    return 0;
}

void orc_free_access(orc_owned_access* a) {
    free(a->z_dim); free(a->x_dim); free(a->y_dim); free(a->y_idx); free(a->xz_end); free(a->level_offset);
    memset(a, 0, sizeof(*a));
}

static double footprint(int l, int iz, int ix, int iy, int glm, const int dims[3]) {
    /* cell_footprint_volume (tree.hpp:15-22) */
    const int s = cell_size(glm, l);
    const int z1 = (iz + 1) * s < dims[0] ? (iz + 1) * s : dims[0];
    const int x1 = (ix + 1) * s < dims[1] ? (ix + 1) * s : dims[1];
    const int y1 = (iy + 1) * s < dims[2] ? (iy + 1) * s : dims[2];
    const double dz = z1 - iz * s, dx = x1 - ix * s, dy = y1 - iy * s;
    return dz * dx * dy;
}

/* One forward merge of child row (l,z,x) against parent row (l-1,z/2,x/2):
 * synchronized_parent_pass (tree.hpp:88-103).  kind 0: leaf child adds
 * w*value; kind 1: tree child adds its own sums. */
static int parent_pass(const orc_access* child, const orc_access* parent, int l, int z, int x, int kind,
                       const float* leaf_values, const int dims[3], int glm, double* vsum, double* wsum) {
    uint64_t rb, re, pb, pe;
    if (orc_get_row(child, l, z, x, &rb, &re)) return -1;
    if (rb == re) return 0;
    if (orc_get_row(parent, l - 1, z / 2, x / 2, &pb, &pe)) return -1;
    uint64_t j = pb;
    for (uint64_t i = rb; i < re; ++i) {
        const int target = child->y_idx[i] / 2;
        while (j < pe && parent->y_idx[j] < target) ++j;
        if (j == pe || parent->y_idx[j] != target) return -3;
        if (kind == 0) {
            const double w = footprint(l, z, x, child->y_idx[i], glm, dims);
            vsum[j] += w * (double)leaf_values[i];
            wsum[j] += w;
        } else {
            vsum[j] += vsum[i];
            wsum[j] += wsum[i];
        }
    }
    return 0;
}

int orc_fill_tree(const orc_access* leaf, const orc_access* tree, const int dims[3], const float* leaf_values,
                  float* tree_out) {
    /* tree.hpp:110-150 */
    const uint64_t nt = tree->n_particles;
    double* vsum = calloc(nt ? nt : 1, sizeof(double));
    double* wsum = calloc(nt ? nt : 1, sizeof(double));
    const int glm = leaf->l_max;
    int st = 0;
    for (int lt = tree->l_max; lt >= tree->l_min && !st; --lt) {
        const int c = lt + 1;
        const int czd = grid_dim(dims[0], glm, c), cxd = grid_dim(dims[1], glm, c);
        for (int pz = 0; pz < tree->z_dim[lt] && !st; ++pz)
            for (int px = 0; px < tree->x_dim[lt] && !st; ++px)
                for (int cz = 2 * pz; cz < 2 * pz + 2 && cz < czd && !st; ++cz)
                    for (int cx = 2 * px; cx < 2 * px + 2 && cx < cxd && !st; ++cx) {
                        if (c >= leaf->l_min && c <= leaf->l_max)
                            st = parent_pass(leaf, tree, c, cz, cx, 0, leaf_values, dims, glm, vsum, wsum);
                        if (!st && c <= tree->l_max)
                            st = parent_pass(tree, tree, c, cz, cx, 1, NULL, dims, glm, vsum, wsum);
                    }
    }
    for (uint64_t i = 0; i < nt; ++i) tree_out[i] = wsum[i] > 0.0 ? (float)(vsum[i] / wsum[i]) : 0.0f;
    free(vsum);
    free(wsum);
    return st;
}

/* --------------------------------------------------------------- index ---- */

int64_t orc_nonempty_rows(const orc_access* a, int level, int* z, int* x, uint16_t* ymin, uint16_t* ymax,
                          int64_t cap) {
    /* convolve.hpp:32-44 */
    int64_t n = 0;
    for (int zz = 0; zz < a->z_dim[level]; ++zz)
        for (int xx = 0; xx < a->x_dim[level]; ++xx) {
            uint64_t b, e;
            orc_get_row(a, level, zz, xx, &b, &e);
            if (b == e) continue;
            if (z && n < cap) {
                z[n] = zz;
                x[n] = xx;
                ymin[n] = a->y_idx[b];
                ymax[n] = a->y_idx[e - 1];
            }
            ++n;
        }
    return n;
}

/* ------------------------------------------------------- reconstruction ---- */

void orc_fill_level_row(const orc_access* leaf, const float* values, const orc_access* tree,
                        const float* tree_values, int l, int z, int x, float* dst, int y_begin, int y_end) {
    /* reconstruct.hpp:41-69: leaves at l-d (d = 0..l-l_min) constant-upsampled
     * by 2^d, then level-l interior nodes. */
    for (int d = 0; d <= l - leaf->l_min; ++d) {
        const int ll = l - d;
        if (ll > leaf->l_max) continue;
        const int cz = z >> d, cx = x >> d;
        if (cz >= leaf->z_dim[ll] || cx >= leaf->x_dim[ll]) continue;
        uint64_t b, e;
        orc_get_row(leaf, ll, cz, cx, &b, &e);
        for (uint64_t i = b; i < e; ++i) {
            const int y0 = leaf->y_idx[i] << d;
            int ya = y0 > y_begin ? y0 : y_begin;
            int yb = y0 + (1 << d);
            if (leaf->y_dim[l] < yb) yb = leaf->y_dim[l];
            if (y_end < yb) yb = y_end;
            for (int y = ya; y < yb; ++y) dst[y] = values[i];
        }
    }
    if (tree_values && l <= tree->l_max && l >= tree->l_min && z < tree->z_dim[l] && x < tree->x_dim[l]) {
        uint64_t b, e;
        orc_get_row(tree, l, z, x, &b, &e);
        for (uint64_t i = b; i < e; ++i) {
            const int y = tree->y_idx[i];
            if (y >= y_begin && y < y_end) dst[y] = tree_values[i];
        }
    }
}

void orc_reconstruct_level(const orc_access* leaf, const float* values, const orc_access* tree,
                           const float* tree_values, int l, float* out) {
    /* reconstruct.hpp:73-84 */
    const int zd = leaf->z_dim[l], xd = leaf->x_dim[l], yd = leaf->y_dim[l];
    memset(out, 0, sizeof(float) * (size_t)zd * xd * yd);
    for (int z = 0; z < zd; ++z)
        for (int x = 0; x < xd; ++x)
            orc_fill_level_row(leaf, values, tree, tree_values, l, z, x, out + ((size_t)z * xd + x) * yd, 0, yd);
}

void orc_reconstruct_patch(const orc_access* leaf, const float* values, const orc_access* tree,
                           const float* tree_values, const int spec[7], float* out) {
    /* reconstruct.hpp:94-129; spec = level, z_begin, z_end, x_begin, x_end, pad,
     * pad_mode (0 Zero, 1 Reflect).  The caller checks the spec. */
    const int l = spec[0], pad = spec[5], zero = spec[6] == 0;
    const int zd = leaf->z_dim[l], xd = leaf->x_dim[l], yd = leaf->y_dim[l];
    const int onz = spec[2] - spec[1] + 2 * pad, onx = spec[4] - spec[3] + 2 * pad, ony = yd + 2 * pad;
    /* one row buffer for the whole patch, as the reference (:108): a cell no
     * source covers keeps the previous row's value */
    float* row = (float*)calloc((size_t)(yd > 0 ? yd : 1), sizeof(float));
    memset(out, 0, sizeof(float) * (size_t)onz * onx * ony);
    for (int oz = 0; oz < onz; ++oz) {
        const int z = spec[1] - pad + oz;
        for (int ox = 0; ox < onx; ++ox) {
            const int x = spec[3] - pad + ox;
            float* dst = out + ((size_t)oz * onx + ox) * ony;
            const int inside = z >= 0 && z < zd && x >= 0 && x < xd;
            if (!inside && zero) continue;
            const int zr = inside ? z : orc_reflect_index(z, zd), xr = inside ? x : orc_reflect_index(x, xd);
            orc_fill_level_row(leaf, values, tree, tree_values, l, zr, xr, row, 0, yd);
            for (int y = 0; y < yd; ++y) dst[pad + y] = row[y];
            for (int p = 0; p < pad; ++p) {
                dst[p] = zero ? 0.0f : row[orc_reflect_index(p - pad, yd)];
                dst[pad + yd + p] = zero ? 0.0f : row[orc_reflect_index(yd + p, yd)];
            }
        }
    }
    free(row);
}

void orc_convolve_pixels(const float* v, int nz, int nx, int ny, const float* w, int kz, int kx, int ky,
                         int pad, float* out) {
    /* convolve.hpp:48-98: pad (reflect_index or zeros) by the half-extents, then
     * per output a double accumulator over (az, ax, ay), zero weights skipped */
    const int hz = kz / 2, hx = kx / 2, hy = ky / 2;
    const int pz = nz + 2 * hz, px = nx + 2 * hx, py = ny + 2 * hy;
    float* padded = (float*)calloc((size_t)pz * px * py, sizeof(float));
    for (int z = 0; z < pz; ++z) {
        const int sz = z - hz, zo = sz < 0 || sz >= nz;
        if (zo && pad == 0) continue;
        const int zr = zo ? orc_reflect_index(sz, nz) : sz;
        for (int x = 0; x < px; ++x) {
            const int sx = x - hx, xo = sx < 0 || sx >= nx;
            if (xo && pad == 0) continue;
            const int xr = xo ? orc_reflect_index(sx, nx) : sx;
            float* dst = padded + ((size_t)z * px + x) * py;
            const float* src = v + ((size_t)zr * nx + xr) * ny;
            memcpy(dst + hy, src, sizeof(float) * (size_t)ny);
            if (pad == 1)
                for (int p = 0; p < hy; ++p) {
                    dst[p] = src[orc_reflect_index(p - hy, ny)];
                    dst[hy + ny + p] = src[orc_reflect_index(ny + p, ny)];
                }
        }
    }
    double* acc = (double*)malloc(sizeof(double) * (size_t)(ny > 0 ? ny : 1));
    for (int z = 0; z < nz; ++z)
        for (int x = 0; x < nx; ++x) {
            for (int y = 0; y < ny; ++y) acc[y] = 0.0;
            for (int az = 0; az < kz; ++az)
                for (int ax = 0; ax < kx; ++ax)
                    for (int ay = 0; ay < ky; ++ay) {
                        const float wv = w[((size_t)az * kx + ax) * ky + ay];
                        if (wv == 0.0f) continue;
                        const float* src = padded + ((size_t)(z + 2 * hz - az) * px + (x + 2 * hx - ax)) * py + (2 * hy - ay);
                        for (int y = 0; y < ny; ++y) acc[y] += (double)wv * (double)src[y];
                    }
            float* dst = out + ((size_t)z * nx + x) * ny;
            for (int y = 0; y < ny; ++y) dst[y] = (float)acc[y];
        }
    free(acc);
    free(padded);
}

/* -------------------------------------------------------------- stencil ---- */

static int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

static int coarse_span(int k, int m) { /* stencil.hpp:131-137 */
    const int h = k / 2;
    const int lo = -((h + m - 1) / m);
    const int hi = (m - 1 + h) / m;
    return -lo > hi ? -lo : hi;
}

void orc_restrict_stencil(const float* w, int kz, int kx, int ky, int delta, int out_k3[3], float* out) {
    /* stencil.hpp:127-160, literally: O(m^3 k^3) with the same accumulation
     * order (oz, ox, oy, rz, rx, ry) into double, one rounding to float. */
    if (delta == 0) {
        out_k3[0] = kz; out_k3[1] = kx; out_k3[2] = ky;
        if (out) memcpy(out, w, sizeof(float) * (size_t)kz * kx * ky);
        return;
    }
    const int m = 1 << delta;
    const int Hz = coarse_span(kz, m), Hx = coarse_span(kx, m), Hy = coarse_span(ky, m);
    const int okz = 2 * Hz + 1, okx = 2 * Hx + 1, oky = 2 * Hy + 1;
    out_k3[0] = okz; out_k3[1] = okx; out_k3[2] = oky;
    if (!out) return;
    double* acc = calloc((size_t)okz * okx * oky, sizeof(double));
    const double inv = 1.0 / ((double)m * m * m);
    const int hz = kz / 2, hx = kx / 2, hy = ky / 2;
    for (int oz = 0; oz < m; ++oz)
        for (int ox = 0; ox < m; ++ox)
            for (int oy = 0; oy < m; ++oy)
                for (int rz = -hz; rz <= hz; ++rz)
                    for (int rx = -hx; rx <= hx; ++rx)
                        for (int ry = -hy; ry <= hy; ++ry) {
                            const int Kz = -floor_div(oz - rz, m);
                            const int Kx = -floor_div(ox - rx, m);
                            const int Ky = -floor_div(oy - ry, m);
                            const float wv = w[((size_t)(rz + hz) * kx + (rx + hx)) * ky + (ry + hy)];
                            acc[((size_t)(Kz + Hz) * okx + (Kx + Hx)) * oky + (Ky + Hy)] += inv * wv;
                        }
    for (size_t i = 0; i < (size_t)okz * okx * oky; ++i) out[i] = (float)acc[i];
    free(acc);
}

/* ----------------------------------------------------------- convolution ---- */

int orc_convolve(const orc_access* leaf, const orc_access* tree, const float* values, const float* tree_values,
                 const orc_pyramid* pyr, int pad, float* out) {
    /* convolve.hpp:220-303.  Each particle at (l,z,x,y) receives
     *   float( sum_{az,ax,ay} double(w_l[az][ax][ay]) * double(I_l(z+hz-az, x+hx-ax, y+hy-ay)) )
     * accumulated from 0.0 in az -> ax -> ay order (LevelSlab::apply,
     * convolve.hpp:154-169), where I_l is the level-l reconstruction
     * (fill_level_row) with per-axis Zero/Reflect padding on the level-l grid
     * (ensure_plane, convolve.hpp:124-150).  Here I_l is materialised densely. */
    if (pyr->l_min > leaf->l_min || pyr->l_max < leaf->l_max) return -1;
    for (int l = leaf->l_min; l <= leaf->l_max; ++l) {
        const int* k = pyr->k3 + 3 * (l - pyr->l_min);
        if (k[0] > ORC_MAX_EXTENT || k[1] > ORC_MAX_EXTENT || k[2] > ORC_MAX_EXTENT) return -2;
    }
    memset(out, 0, sizeof(float) * leaf->n_particles);
    for (int l = leaf->l_min; l <= leaf->l_max; ++l) {
        const int zd = leaf->z_dim[l], xd = leaf->x_dim[l], yd = leaf->y_dim[l];
        uint64_t lb, le;
        {
            uint64_t r0 = leaf->level_offset[l], r1 = r0 + (uint64_t)zd * xd;
            lb = r0 ? leaf->xz_end[r0 - 1] : 0;
            le = r1 ? leaf->xz_end[r1 - 1] : 0;
        }
        if (lb == le) continue;
        const int* k = pyr->k3 + 3 * (l - pyr->l_min);
        const int kz = k[0], kx = k[1], ky = k[2];
        const int hz = kz / 2, hx = kx / 2, hy = ky / 2;
        const float* w = pyr->w + pyr->off[l - pyr->l_min];
        float* img = malloc(sizeof(float) * ((size_t)zd * xd * yd + 1));
        orc_reconstruct_level(leaf, values, tree, tree_values, l, img);
        for (int z = 0; z < zd; ++z)
            for (int x = 0; x < xd; ++x) {
                uint64_t b, e;
                orc_get_row(leaf, l, z, x, &b, &e);
                for (uint64_t i = b; i < e; ++i) {
                    const int y = leaf->y_idx[i];
                    double acc = 0.0;
                    for (int az = 0; az < kz; ++az) {
                        int zs = z + hz - az;
                        const int zo = zs < 0 || zs >= zd;
                        if (zo) zs = orc_reflect_index(zs, zd);
                        for (int ax = 0; ax < kx; ++ax) {
                            int xs = x + hx - ax;
                            const int xo = xs < 0 || xs >= xd;
                            if (xo) xs = orc_reflect_index(xs, xd);
                            const float* row = img + ((size_t)zs * xd + xs) * yd;
                            const float* wr = w + ((size_t)az * kx + ax) * ky;
                            for (int ay = 0; ay < ky; ++ay) {
                                int ys = y + hy - ay;
                                const int yo = ys < 0 || ys >= yd;
                                if (yo) ys = orc_reflect_index(ys, yd);
                                const float u = (pad == 0 && (zo || xo || yo)) ? 0.0f : row[ys];
                                acc += (double)wr[ay] * (double)u;
                            }
                        }
                    }
                    out[i] = (float)acc;
                }
            }
        free(img);
    }
    return 0;
}

/* ------------------------------------------------------------------- RL ---- */

int orc_rl_apr(const orc_access* leaf, const orc_access* tree, const int dims[3], const float* observed,
               const orc_pyramid* pyr_w, const orc_pyramid* pyr_wt, int iterations, double eps, float* out) {
    /* deconv.hpp:75-107 (pyramids and eps prepared by the caller, :79-93) */
    const uint64_t n = leaf->n_particles, nt = tree->n_particles;
    float* u = malloc(sizeof(float) * (n ? n : 1));
    float* ratio = malloc(sizeof(float) * (n ? n : 1));
    float* tmp = malloc(sizeof(float) * (n ? n : 1));
    float* tv = malloc(sizeof(float) * (nt ? nt : 1));
    for (uint64_t i = 0; i < n; ++i) u[i] = observed[i] > 0.0f ? observed[i] : 0.0f; /* std::max(v, 0.0f) */
    memcpy(out, u, sizeof(float) * n);
    int st = 0;
    for (int k = 1; k <= iterations && !st; ++k) {
        st = orc_fill_tree(leaf, tree, dims, out, tv);
        if (!st) st = orc_convolve(leaf, tree, out, tv, pyr_w, 1, tmp);
        for (uint64_t i = 0; i < n && !st; ++i) {
            const double b = (double)tmp[i];
            const double d = b < eps ? eps : b; /* std::max<double>(blurred, eps) */
            ratio[i] = (float)((double)u[i] / d);
        }
        if (!st) st = orc_fill_tree(leaf, tree, dims, ratio, tv);
        if (!st) st = orc_convolve(leaf, tree, ratio, tv, pyr_wt, 1, tmp);
        for (uint64_t i = 0; i < n && !st; ++i) out[i] *= tmp[i];
    }
    free(u); free(ratio); free(tmp); free(tv);
    return st;
}

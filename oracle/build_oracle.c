/* oracle/build_oracle.c -- TEST INFRASTRUCTURE ONLY (never linked by the
 * product; used by tests/ and by bench.py's reference arm / cpu_baseline to
 * make their inputs without touching the GPU library).
 *
 * A multi-threaded plain-C restatement of the reference's input side for the
 * synthetic sphere workloads (BASELINE configs C1-C5):
 *   generate_spheres   synthetic.hpp:74-111 (separable_gaussian :34-67)
 *   build_apr          build.hpp:290-312 with SigmaPolicy::constant(intensity
 *                      range), central-difference gradient, no smoothing:
 *     gradient_magnitude :42-75 -> level_function :113-129 -> +1 safety
 *     level :301-303 -> solve_levels :136-248 -> sample_particles :252-284
 * Every floating-point step keeps the reference's operation order (compiled
 * with -ffp-contract=off, like the reference oracle), so the structure and the
 * sampled values are bit-identical to the reference build -- pinned by
 * tests/test_oracle.py against the live reference (oracle/_ref) and the
 * committed golden C1 fixture.  Parallel over z planes / cells only where
 * the reference's result does not depend on the visiting order (every output
 * element is computed by one thread in the reference's per-element order).
 * Memory: ~10 GB at 1024^3 (the reference peaks at 34 GB).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "aprk_oracle.h"

/* ---- a tiny static-chunked parallel for ------------------------------------ */
typedef void (*orc_body)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
    orc_body f;
    void* ctx;
    int64_t n, chunk;
    int64_t next;
    pthread_mutex_t mu;
} orc_pf;

static void* pf_worker(void* arg) {
    orc_pf* p = (orc_pf*)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        const int64_t lo = p->next;
        p->next += p->chunk;
        pthread_mutex_unlock(&p->mu);
        if (lo >= p->n) return NULL;
        p->f(p->ctx, lo, lo + p->chunk < p->n ? lo + p->chunk : p->n);
    }
}

static int g_threads = 1;

static void parallel_for(int64_t n, int64_t chunk, orc_body f, void* ctx) {
    if (n <= 0) return;
    orc_pf p;
    p.f = f;
    p.ctx = ctx;
    p.n = n;
    p.chunk = chunk < 1 ? 1 : chunk;
    p.next = 0;
    pthread_mutex_init(&p.mu, NULL);
    int nt = g_threads;
    if (nt > 256) nt = 256;
    pthread_t th[256];
    int started = 0;
    for (int i = 1; i < nt; ++i)
        if (pthread_create(&th[started], NULL, pf_worker, &p) == 0) ++started;
    pf_worker(&p);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&p.mu);
}

/* ---- CounterRng (rng.hpp:8-55) --------------------------------------------- */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
typedef struct {
    uint64_t seed, counter;
} crng;
static double rng_double(crng* r) {
    const uint64_t u = splitmix64(r->seed ^ splitmix64(r->counter++));
    return (double)(u >> 11) * 0x1.0p-53;
}
static double rng_uniform(crng* r, double lo, double hi) { return lo + (hi - lo) * rng_double(r); }

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* ---- generate_spheres -------------------------------------------------------- */
typedef struct {
    float* v;
    int nz, nx, ny;
    double cz, cx, cy, r2;
    float val;
    int z0, x0, x1, y0, y1;
} sph_ctx;

static void sph_body(void* c, int64_t lo, int64_t hi) {
    sph_ctx* s = (sph_ctx*)c;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = s->z0 + (int)zi;
        for (int x = s->x0; x <= s->x1; ++x)
            for (int y = s->y0; y <= s->y1; ++y) {
                const double dz = z - s->cz, dx = x - s->cx, dy = y - s->cy;
                if (dz * dz + dx * dx + dy * dy <= s->r2)
                    s->v[((size_t)z * s->nx + x) * s->ny + y] = s->val;
            }
    }
}

typedef struct {
    const float* in;
    float* out;
    int nz, nx, ny, axis, h;
    const double* g;
} blur_ctx;

static int reflect_i(int i, int n) {  /* separable_gaussian's reflect (synthetic.hpp:46-49) */
    while (i < 0 || i >= n) i = i < 0 ? -i - 1 : 2 * n - 1 - i;
    return i;
}

/* one axis of separable_gaussian (synthetic.hpp:60-66).  Every output keeps
 * the reference's per-element order -- acc from 0, taps i = -h..h, each
 * acc += g * value -- while the loops run over whole y rows (vectorised across
 * elements, never within one element's sum). */
static void blur_body(void* c, int64_t lo, int64_t hi) {
    blur_ctx* b = (blur_ctx*)c;
    const int nx = b->nx, ny = b->ny, h = b->h;
    double* acc = (double*)malloc(sizeof(double) * (size_t)ny);
    if (!acc) abort();
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        for (int x = 0; x < nx; ++x) {
            float* out = b->out + ((size_t)z * nx + x) * ny;
            for (int y = 0; y < ny; ++y) acc[y] = 0.0;
            if (b->axis < 2) {
                for (int i = -h; i <= h; ++i) {
                    const int zz = b->axis == 0 ? reflect_i(z + i, b->nz) : z;
                    const int xx = b->axis == 1 ? reflect_i(x + i, nx) : x;
                    const float* row = b->in + ((size_t)zz * nx + xx) * ny;
                    const double g = b->g[i + h];
                    for (int y = 0; y < ny; ++y) acc[y] += g * row[y];
                }
            } else {
                const float* row = b->in + ((size_t)z * nx + x) * ny;
                for (int i = -h; i <= h; ++i) {
                    const double g = b->g[i + h];
                    const int ylo = h < ny ? h : ny, yhi = ny - h > ylo ? ny - h : ylo;
                    for (int y = 0; y < ylo; ++y) acc[y] += g * row[reflect_i(y + i, ny)];
                    for (int y = ylo; y < yhi; ++y) acc[y] += g * row[y + i];
                    for (int y = yhi; y < ny; ++y) acc[y] += g * row[reflect_i(y + i, ny)];
                }
            }
            for (int y = 0; y < ny; ++y) out[y] = (float)acc[y];
        }
    }
    free(acc);
}

int orc_generate_spheres(int nz, int nx, int ny, int count, double min_r, double max_r, double background,
                         double min_i, double max_i, double blur, uint64_t seed, int threads, float* v) {
    g_threads = threads > 0 ? threads : 1;
    crng r = {seed, 0};
    const size_t n = (size_t)nz * nx * ny;
    const float bg = (float)background;
    for (size_t i = 0; i < n; ++i) v[i] = bg;
    for (int k = 0; k < count; ++k) { /* synthetic.hpp:76-83, then :86-100 in sphere order */
        const double rad = rng_uniform(&r, min_r, max_r);
        const double cz = rng_uniform(&r, rad, fmax(nz - rad, rad));
        const double cx = rng_uniform(&r, rad, fmax(nx - rad, rad));
        const double cy = rng_uniform(&r, rad, fmax(ny - rad, rad));
        const double inten = rng_uniform(&r, min_i, max_i);
        /* the RNG draws all spheres first (the reference fills `spheres` before
         * drawing), so drawing and rasterising interleaved is the same stream */
        sph_ctx s;
        s.v = v;
        s.nz = nz;
        s.nx = nx;
        s.ny = ny;
        s.cz = cz;
        s.cx = cx;
        s.cy = cy;
        s.r2 = rad * rad;
        s.val = (float)inten;
        s.z0 = imax(0, (int)floor(cz - rad));
        const int z1 = imin(nz - 1, (int)ceil(cz + rad));
        s.x0 = imax(0, (int)floor(cx - rad));
        s.x1 = imin(nx - 1, (int)ceil(cx + rad));
        s.y0 = imax(0, (int)floor(cy - rad));
        s.y1 = imin(ny - 1, (int)ceil(cy + rad));
        parallel_for(z1 - s.z0 + 1, 1, sph_body, &s);
    }
    if (blur > 0.0) {
        const int size = 2 * (int)ceil(3.0 * blur) + 1, h = size / 2;
        double* g = (double*)malloc(sizeof(double) * size);
        if (!g) return -1;
        double norm = 0.0;
        for (int i = -h; i <= h; ++i) {
            g[i + h] = exp(-0.5 * i * i / (blur * blur));
            norm += g[i + h];
        }
        for (int i = 0; i < size; ++i) g[i] /= norm;
        float* tmp = (float*)malloc(sizeof(float) * n);
        if (!tmp) {
            free(g);
            return -1;
        }
        for (int axis = 0; axis < 3; ++axis) { /* PixelVolume tmp = v; v.at = blur(tmp) */
            memcpy(tmp, v, sizeof(float) * n);
            blur_ctx b = {tmp, v, nz, nx, ny, axis, h, g};
            parallel_for(nz, 1, blur_body, &b);
        }
        free(tmp);
        free(g);
    }
    return 0;
}

/* ---- build_apr (spheres recipe) ---------------------------------------------- */
static int grid_dim(int n, int l_max, int l) { /* linear_access.hpp:21-24 */
    const int s = 1 << (l_max - l);
    return (n + s - 1) / s;
}

typedef struct {
    int zd, xd, yd;
} g3;
static size_t g3n(g3 g) { return (size_t)g.zd * g.xd * g.yd; }

typedef struct {
    const float* v;
    int8_t* T;
    int nz, nx, ny, l_min, l_max;
    double E, sigma, omega;
} tgt_ctx;

static void tgt_body(void* c, int64_t lo, int64_t hi) {
    tgt_ctx* t = (tgt_ctx*)c;
    const int nz = t->nz, nx = t->nx, ny = t->ny;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        const int zp = imin(z + 1, nz - 1), zm = imax(z - 1, 0);
        for (int x = 0; x < nx; ++x) {
            const int xp = imin(x + 1, nx - 1), xm = imax(x - 1, 0);
            for (int y = 0; y < ny; ++y) {
                const int yp = imin(y + 1, ny - 1), ym = imax(y - 1, 0);
#define AT(a, b, d) t->v[((size_t)(a) * nx + (b)) * ny + (d)]
                const float dzf = AT(zp, x, y) - AT(zm, x, y); /* float - float, then 0.5 * double */
                const float dxf = AT(z, xp, y) - AT(z, xm, y);
                const float dyf = AT(z, x, yp) - AT(z, x, ym);
#undef AT
                const double gz = 0.5 * dzf, gx = 0.5 * dxf, gy = 0.5 * dyf;
                const float g = (float)sqrt(gz * gz + gx * gx + gy * gy); /* gradient_magnitude, :70 */
                int lev;
                if ((double)g <= 0.0) {
                    lev = t->l_min;
                } else { /* level_function, :121-125 */
                    const double L = t->E * t->sigma / (double)g;
                    const int l = (int)ceil(log2(t->omega / L));
                    lev = imin(imax(l, t->l_min), t->l_max);
                }
                lev = imin(lev + 1, t->l_max); /* constant-sigma safety level, :301-303 */
                t->T[((size_t)z * nx + x) * ny + y] = (int8_t)imin(imax(lev, t->l_min), t->l_max); /* :172 */
            }
        }
    }
}

typedef struct {
    const int8_t* f;
    int8_t* c;
    g3 fg, cg;
} mr_ctx;

static void mr_body(void* cc, int64_t lo, int64_t hi) { /* max_reduce, :158-166, as a gather */
    mr_ctx* m = (mr_ctx*)cc;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        for (int x = 0; x < m->cg.xd; ++x)
            for (int y = 0; y < m->cg.yd; ++y) {
                int mx = 0;
                for (int a = 2 * z; a < imin(2 * z + 2, m->fg.zd); ++a)
                    for (int b = 2 * x; b < imin(2 * x + 2, m->fg.xd); ++b)
                        for (int d = 2 * y; d < imin(2 * y + 2, m->fg.yd); ++d) {
                            const int v = m->f[((size_t)a * m->fg.xd + b) * m->fg.yd + d];
                            if (v > mx) mx = v;
                        }
                m->c[((size_t)z * m->cg.xd + x) * m->cg.yd + y] = (int8_t)mx;
            }
    }
}

typedef struct {
    const int8_t* T;
    const uint8_t* fine;
    uint8_t* need;
    g3 g, fg;
    int l;
} need_ctx;

static void need_body(void* cc, int64_t lo, int64_t hi) { /* :176-203 as a gather */
    need_ctx* q = (need_ctx*)cc;
    const g3 g = q->g, fg = q->fg;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        for (int x = 0; x < g.xd; ++x)
            for (int y = 0; y < g.yd; ++y) {
                const size_t i = ((size_t)z * g.xd + x) * g.yd + y;
                uint8_t r = q->T[i] >= q->l ? 1 : 0;
                if (!r && q->fine) {
                    const int pz1 = imin(2 * z + 1, fg.zd - 1), px1 = imin(2 * x + 1, fg.xd - 1),
                              py1 = imin(2 * y + 1, fg.yd - 1);
                    for (int a = imax(2 * z - 1, 0); a <= imin(pz1 + 1, fg.zd - 1) && !r; ++a)
                        for (int b = imax(2 * x - 1, 0); b <= imin(px1 + 1, fg.xd - 1) && !r; ++b)
                            for (int d = imax(2 * y - 1, 0); d <= imin(py1 + 1, fg.yd - 1); ++d)
                                if (q->fine[((size_t)a * fg.xd + b) * fg.yd + d]) {
                                    r = 1;
                                    break;
                                }
                }
                q->need[i] = r;
            }
    }
}

typedef struct {
    uint8_t** need;
    g3* g;
    int8_t* G;
    g3 pg;
    int l_min, l_max;
} fd_ctx;

static void fd_body(void* cc, int64_t lo, int64_t hi) { /* :205-223: finest demand per pixel */
    fd_ctx* f = (fd_ctx*)cc;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        for (int x = 0; x < f->pg.xd; ++x)
            for (int y = 0; y < f->pg.yd; ++y) {
                int e = f->l_min;
                for (int l = f->l_max; l > f->l_min; --l) {
                    const int d = f->l_max - l;
                    const g3 g = f->g[l];
                    if (f->need[l][((size_t)(z >> d) * g.xd + (x >> d)) * g.yd + (y >> d)]) {
                        e = l;
                        break;
                    }
                }
                f->G[((size_t)z * f->pg.xd + x) * f->pg.yd + y] = (int8_t)e;
            }
    }
}

typedef struct {
    const int8_t* gl;
    const int8_t* gp;
    g3 g, pg;
    int l, l_min;
    uint64_t* counts; /* per row (pass 0) */
    const uint64_t* begin; /* per row (pass 1) */
    uint16_t* y_out;
    int pass;
} leaf_ctx;

static void leaf_body(void* cc, int64_t lo, int64_t hi) { /* :228-246 */
    leaf_ctx* c = (leaf_ctx*)cc;
    const g3 g = c->g, pg = c->pg;
    for (int64_t r = lo; r < hi; ++r) {
        const int z = (int)(r / g.xd), x = (int)(r % g.xd);
        uint64_t pos = c->pass ? c->begin[r] : 0, cnt = 0;
        for (int y = 0; y < g.yd; ++y) {
            if (c->gl[((size_t)z * g.xd + x) * g.yd + y] > c->l) continue;
            if (c->l > c->l_min && c->gp[((size_t)(z >> 1) * pg.xd + (x >> 1)) * pg.yd + (y >> 1)] <= c->l - 1)
                continue;
            if (c->pass) c->y_out[pos++] = (uint16_t)y;
            ++cnt;
        }
        if (!c->pass) c->counts[r] = cnt;
    }
}

typedef struct {
    const float* vf;
    const double* fs;
    double* cs;
    g3 fg, cg;
} sum_ctx;

static void sum_body(void* cc, int64_t lo, int64_t hi) { /* sample_particles' pyramid, :262-274 */
    sum_ctx* s = (sum_ctx*)cc;
    for (int64_t zi = lo; zi < hi; ++zi) {
        const int z = (int)zi;
        for (int x = 0; x < s->cg.xd; ++x)
            for (int y = 0; y < s->cg.yd; ++y) {
                double acc = 0.0; /* children in the fine grid's (z, x, y) visiting order */
                for (int a = 2 * z; a < imin(2 * z + 2, s->fg.zd); ++a)
                    for (int b = 2 * x; b < imin(2 * x + 2, s->fg.xd); ++b)
                        for (int d = 2 * y; d < imin(2 * y + 2, s->fg.yd); ++d) {
                            const size_t fi = ((size_t)a * s->fg.xd + b) * s->fg.yd + d;
                            acc += s->vf ? (double)s->vf[fi] : s->fs[fi];
                        }
                s->cs[((size_t)z * s->cg.xd + x) * s->cg.yd + y] = acc;
            }
    }
}

typedef struct {
    const orc_owned_access* a;
    double** S;
    g3* g;
    const float* vol;
    int nz, nx, ny, l;
    float* out;
} samp_ctx;

static void samp_body(void* cc, int64_t lo, int64_t hi) { /* :276-283 */
    samp_ctx* c = (samp_ctx*)cc;
    const orc_owned_access* a = c->a;
    const int l = c->l, lm = a->l_max, s = 1 << (lm - l);
    for (int64_t r = lo; r < hi; ++r) {
        const int z = (int)(r / a->x_dim[l]), x = (int)(r % a->x_dim[l]);
        const uint64_t row = a->level_offset[l] + (uint64_t)r;
        const uint64_t b = row ? a->xz_end[row - 1] : 0, e = a->xz_end[row];
        for (uint64_t i = b; i < e; ++i) {
            const int y = a->y_idx[i];
            if (l == lm) {
                c->out[i] = (float)((double)c->vol[((size_t)z * c->nx + x) * c->ny + y] / 1.0);
            } else {
                const g3 g = c->g[l];
                const double sum = c->S[l][((size_t)z * g.xd + x) * g.yd + y];
                /* the weight pyramid sums 1.0s: the clipped footprint, exactly */
                const double wz = imin((z + 1) * s, c->nz) - z * s, wx = imin((x + 1) * s, c->nx) - x * s,
                             wy = imin((y + 1) * s, c->ny) - y * s;
                c->out[i] = (float)(sum / (wz * wx * wy));
            }
        }
    }
}

static int compute_l_max(int nz, int nx, int ny) { /* linear_access.hpp:27-32 */
    const int m = imax(nz, imax(nx, ny));
    int l = 0;
    while ((1 << l) < m) ++l;
    return l;
}

int orc_build_apr(const float* v, int nz, int nx, int ny, double rel_error, int threads, orc_owned_access* out,
                  float** values_out) {
    g_threads = threads > 0 ? threads : 1;
    memset(out, 0, sizeof(*out));
    *values_out = NULL;
    if (nz < 1 || nx < 1 || ny < 1 || ny > 65536) return -1;
    const int l_max = compute_l_max(nz, nx, ny), l_min = imin(1, l_max);
    if (l_max >= 24) return -1;
    const size_t n = (size_t)nz * nx * ny;
    g3 gd[24];
    for (int l = 0; l <= l_max; ++l) gd[l] = (g3){grid_dim(nz, l_max, l), grid_dim(nx, l_max, l), grid_dim(ny, l_max, l)};
    /* intensity_range -> constant sigma = float(max(range, floor)) (build.hpp:80-86) */
    float mn = v[0], mx = v[0];
    for (size_t i = 1; i < n; ++i) {
        if (v[i] < mn) mn = v[i];
        if (v[i] > mx) mx = v[i];
    }
    const float range = mx - mn;
    const double floor_value = 1e-3 * (double)(1e-30f > range ? 1e-30f : range);
    const double sigma = (double)(float)((double)range > floor_value ? (double)range : floor_value);

    int8_t* T[24] = {0};
    uint8_t* need[24] = {0};
    int8_t* Gm[24] = {0};
    T[l_max] = (int8_t*)malloc(n);
    if (!T[l_max]) return -1;
    tgt_ctx tc = {v, T[l_max], nz, nx, ny, l_min, l_max, rel_error, sigma, (double)(1u << l_max)};
    parallel_for(nz, 1, tgt_body, &tc);
    for (int l = l_max - 1; l >= l_min; --l) {
        T[l] = (int8_t*)malloc(g3n(gd[l]) + 1);
        mr_ctx m = {T[l + 1], T[l], gd[l + 1], gd[l]};
        parallel_for(gd[l].zd, 1, mr_body, &m);
    }
    for (int l = l_max; l >= l_min; --l) {
        need[l] = (uint8_t*)malloc(g3n(gd[l]) + 1);
        need_ctx q = {T[l], l < l_max ? need[l + 1] : NULL, need[l], gd[l], l < l_max ? gd[l + 1] : gd[l], l};
        parallel_for(gd[l].zd, 1, need_body, &q);
    }
    for (int l = l_min; l <= l_max; ++l) free(T[l]);
    Gm[l_max] = (int8_t*)malloc(n);
    fd_ctx f = {need, gd, Gm[l_max], gd[l_max], l_min, l_max};
    parallel_for(nz, 1, fd_body, &f);
    for (int l = l_min; l <= l_max; ++l) free(need[l]);
    for (int l = l_max - 1; l >= l_min; --l) {
        Gm[l] = (int8_t*)malloc(g3n(gd[l]) + 1);
        mr_ctx m = {Gm[l + 1], Gm[l], gd[l + 1], gd[l]};
        parallel_for(gd[l].zd, 1, mr_body, &m);
    }
    /* leaf rows -> CSR (assemble_access, linear_access.hpp:101-130) */
    out->l_min = l_min;
    out->l_max = l_max;
    out->z_dim = (int*)calloc(l_max + 1, sizeof(int));
    out->x_dim = (int*)calloc(l_max + 1, sizeof(int));
    out->y_dim = (int*)calloc(l_max + 1, sizeof(int));
    out->level_offset = (uint64_t*)calloc(l_max + 1, sizeof(uint64_t));
    uint64_t rows = 0;
    for (int l = l_min; l <= l_max; ++l) {
        out->z_dim[l] = gd[l].zd;
        out->x_dim[l] = gd[l].xd;
        out->y_dim[l] = gd[l].yd;
        out->level_offset[l] = rows;
        rows += (uint64_t)gd[l].zd * gd[l].xd;
    }
    out->n_rows = rows;
    out->xz_end = (uint64_t*)malloc(sizeof(uint64_t) * (rows + 1));
    uint64_t* begin = (uint64_t*)malloc(sizeof(uint64_t) * (rows + 1));
    for (int pass = 0; pass < 2; ++pass) {
        for (int l = l_min; l <= l_max; ++l) {
            const uint64_t r0 = out->level_offset[l];
            leaf_ctx c = {Gm[l], l > l_min ? Gm[l - 1] : NULL, gd[l], l > l_min ? gd[l - 1] : gd[l], l, l_min,
                          out->xz_end + r0, begin + r0, out->y_idx, pass};
            parallel_for((int64_t)gd[l].zd * gd[l].xd, 256, leaf_body, &c);
        }
        if (pass == 0) {
            uint64_t acc = 0;
            for (uint64_t r = 0; r < rows; ++r) {
                begin[r] = acc;
                acc += out->xz_end[r];
                out->xz_end[r] = acc;
            }
            out->n_particles = acc;
            out->y_idx = (uint16_t*)malloc(2 * acc + 2);
        }
    }
    free(begin);
    for (int l = l_min; l <= l_max; ++l) free(Gm[l]);
    /* sample_particles */
    double* S[24] = {0};
    for (int l = l_max - 1; l >= l_min; --l) {
        S[l] = (double*)malloc(sizeof(double) * g3n(gd[l]) + 8);
        sum_ctx sc = {l == l_max - 1 ? v : NULL, l == l_max - 1 ? NULL : S[l + 1], S[l], gd[l + 1], gd[l]};
        parallel_for(gd[l].zd, 1, sum_body, &sc);
    }
    float* vals = (float*)malloc(sizeof(float) * out->n_particles + 4);
    for (int l = l_min; l <= l_max; ++l) {
        samp_ctx c = {out, S, gd, v, nz, nx, ny, l, vals};
        parallel_for((int64_t)gd[l].zd * gd[l].xd, 256, samp_body, &c);
    }
    for (int l = l_min; l <= l_max; ++l) free(S[l]);
    *values_out = vals;
    return 0;
}

void orc_free_values(float* v) { free(v); }

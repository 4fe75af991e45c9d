/*
 * apbf_oracle.c -- TEST INFRASTRUCTURE ONLY (see apbf_oracle.h).
 *
 * Plain-C float32 restatement of the reference APBF step.  Each function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj/include/apbf/).  Build with -ffp-contract=off and no
 * -march flags so that no FMA contraction happens.
 */
#define _POSIX_C_SOURCE 199309L
#include "apbf_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef float R;

#define PI_F 3.14159265358979323846f
#define K_MAX_CELLS ((int64_t)1 << 26) /* uniform_grid.hpp:40 */

/* ------------------------------------------------------------------ errors */

static int32_t set_err(apbf_error* err, int32_t code, const char* pass, int32_t particle,
                       const char* fmt, ...) {
    if (err) {
        err->code = code;
        err->particle = particle;
        snprintf(err->pass, sizeof err->pass, "%s", pass ? pass : "");
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err->message, sizeof err->message, fmt, ap);
        va_end(ap);
    }
    return code;
}

/* NumericalError what() text (types.hpp:27-29). */
static int32_t numerical(apbf_error* err, const char* pass, int32_t particle, const char* detail) {
    return set_err(err, APBF_ERR_NUMERICAL, pass, particle,
                   "numerical abort in pass '%s' at particle %d: %s", pass, particle, detail);
}

static void clear_err(apbf_error* err) {
    if (err) memset(err, 0, sizeof *err);
}

/* ------------------------------------------------------- Eigen Vec3 order */
/* Fixed-size-3 float reductions unroll as x0 + (x1 + x2) (Eigen's
 * redux_novec_unroller splits the range in halves). */
static inline R sqn3(const R* a) { return a[0] * a[0] + (a[1] * a[1] + a[2] * a[2]); }
static inline R dot3(const R* a, const R* b) { return a[0] * b[0] + (a[1] * b[1] + a[2] * b[2]); }
static inline R norm3(const R* a) { return sqrtf(sqn3(a)); }
static inline R maxf_std(R a, R b) { return (a < b) ? b : a; } /* std::max */
static inline R minf_std(R a, R b) { return (b < a) ? b : a; } /* std::min */
static inline int maxi_std(int a, int b) { return (a < b) ? b : a; }
static inline int mini_std(int a, int b) { return (b < a) ? b : a; }
static inline R clampf_std(R v, R lo, R hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }
static inline int all_finite3(const R* a) {
    return isfinite(a[0]) && isfinite(a[1]) && isfinite(a[2]);
}
static inline void cross3(const R* a, const R* b, R* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

/* ---------------------------------------------------------- SPH kernels */

/* densityKernelR2 (kernels.hpp:38-48). */
float orc_density_kernel_r2(float r2, float h) {
    const R h2 = h * h;
    if (r2 >= h2) return 0.0f;
    const R d = h2 - r2;
    const R h4 = h2 * h2;
    const R norm = 4.921875f / (PI_F * h4 * h4 * h);
    return norm * d * d * d;
}

/* gradientKernel (kernels.hpp:52-65); h > 0 is validated by the callers. */
void orc_gradient_kernel(const float r[3], float h, float out[3]) {
    const R rn = norm3(r);
    if (rn >= h || rn == 0.0f) {
        out[0] = out[1] = out[2] = 0.0f;
        return;
    }
    const R a = h - rn;
    const R h3 = h * h * h;
    const R coeff = -45.0f / (PI_F * h3 * h3) * a * a / rn;
    out[0] = coeff * r[0];
    out[1] = coeff * r[1];
    out[2] = coeff * r[2];
}

/* ------------------------------------------------------------- SDF scene */

typedef struct {
    apbf_sdf_primitive* prims;
    int n;
    R step;
} scene_t;

/* Constructor validation (sdf.hpp:23-29, 38-43, 52-57, 68-73). */
static int32_t scene_init(scene_t* sc, const apbf_sdf_primitive* prims, int n, R step,
                          apbf_error* err) {
    sc->n = n;
    sc->step = step;
    sc->prims = NULL;
    if (n < 0) return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "negative primitive count");
    if (n == 0) return APBF_OK;
    sc->prims = (apbf_sdf_primitive*)malloc(sizeof(apbf_sdf_primitive) * (size_t)n);
    for (int k = 0; k < n; ++k) {
        apbf_sdf_primitive p = prims[k];
        switch (p.kind) {
            case APBF_SDF_HALF_SPACE: {
                const R len = norm3(p.p);
                if (!(len > 0.0f)) {
                    free(sc->prims);
                    sc->prims = NULL;
                    return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                                   "half-space normal must be nonzero");
                }
                p.p[0] /= len;
                p.p[1] /= len;
                p.p[2] /= len;
                break;
            }
            case APBF_SDF_SPHERE:
                if (!(p.a > 0.0f)) {
                    free(sc->prims);
                    sc->prims = NULL;
                    return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                                   "sphere radius must be positive");
                }
                break;
            case APBF_SDF_BOX: {
                /* halfExtents.minCoeff() > 0 */
                const R m = minf_std(p.q[0], minf_std(p.q[1], p.q[2]));
                if (!(m > 0.0f)) {
                    free(sc->prims);
                    sc->prims = NULL;
                    return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                                   "box half extents must be positive");
                }
                break;
            }
            case APBF_SDF_CONE:
                if (!(p.a > 0.0f) || !(p.b > 0.0f)) {
                    free(sc->prims);
                    sc->prims = NULL;
                    return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                                   "cone radius and height must be positive");
                }
                break;
            default:
                free(sc->prims);
                sc->prims = NULL;
                return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "unknown primitive kind");
        }
        sc->prims[k] = p;
    }
    return APBF_OK;
}

/* primitiveDistance(Cone) (sdf.hpp:124-142). */
static R cone_distance(const apbf_sdf_primitive* c, const R* p) {
    const R rho = hypotf(p[0] - c->p[0], p[2] - c->p[2]);
    const R y = p[1] - c->p[1];
    const R Rr = c->a;
    const R H = c->b;
    const R baseDx = rho - clampf_std(rho, 0.0f, Rr);
    const R dBase = hypotf(baseDx, y);
    const R ex = -Rr, ey = H;
    const R t = clampf_std(((rho - Rr) * ex + y * ey) / (ex * ex + ey * ey), 0.0f, 1.0f);
    const R dSlant = hypotf(rho - (Rr + t * ex), y - t * ey);
    const int inside = y >= 0.0f && y <= H && rho <= Rr * (1.0f - y / H);
    const R d = minf_std(dBase, dSlant);
    return inside ? -d : d;
}

/* primitiveDistance (sdf.hpp:102-142). */
static R prim_distance(const apbf_sdf_primitive* pr, const R* p) {
    switch (pr->kind) {
        case APBF_SDF_HALF_SPACE:
            return dot3(pr->p, p) - pr->a;
        case APBF_SDF_SPHERE: {
            R d3[3] = {p[0] - pr->p[0], p[1] - pr->p[1], p[2] - pr->p[2]};
            const R d = norm3(d3) - pr->a;
            return pr->interior ? -d : d;
        }
        case APBF_SDF_BOX: {
            R q[3], qm[3];
            for (int a = 0; a < 3; ++a) {
                q[a] = fabsf(p[a] - pr->p[a]) - pr->q[a];
                qm[a] = maxf_std(q[a], 0.0f);
            }
            const R outside = norm3(qm);
            const R qmax = maxf_std(q[0], maxf_std(q[1], q[2]));
            const R inside = minf_std(qmax, 0.0f);
            const R d = outside + inside;
            return pr->interior ? -d : d;
        }
        default:
            return cone_distance(pr, p);
    }
}

/* primitiveGradient (sdf.hpp:144-196). */
static void prim_gradient(const apbf_sdf_primitive* pr, const R* p, R step, R* g) {
    switch (pr->kind) {
        case APBF_SDF_HALF_SPACE:
            g[0] = pr->p[0];
            g[1] = pr->p[1];
            g[2] = pr->p[2];
            return;
        case APBF_SDF_SPHERE: {
            R d[3] = {p[0] - pr->p[0], p[1] - pr->p[1], p[2] - pr->p[2]};
            const R len = norm3(d);
            if (len <= 0.0f) {
                g[0] = 0.0f;
                g[1] = 1.0f;
                g[2] = 0.0f;
                return;
            }
            d[0] /= len;
            d[1] /= len;
            d[2] /= len;
            for (int a = 0; a < 3; ++a) g[a] = pr->interior ? -d[a] : d[a];
            return;
        }
        case APBF_SDF_BOX: {
            R rel[3], sgn[3], q[3];
            for (int a = 0; a < 3; ++a) {
                rel[a] = p[a] - pr->p[a];
                sgn[a] = rel[a] < 0.0f ? -1.0f : 1.0f;
                q[a] = fabsf(rel[a]) - pr->q[a];
            }
            R gg[3];
            if (maxf_std(q[0], maxf_std(q[1], q[2])) > 0.0f) {
                for (int a = 0; a < 3; ++a) gg[a] = sgn[a] * maxf_std(q[a], 0.0f);
                const R z = sqn3(gg);
                if (z > 0.0f) {
                    const R s = sqrtf(z);
                    gg[0] /= s;
                    gg[1] /= s;
                    gg[2] /= s;
                }
            } else {
                int axis = 0; /* maxCoeff(&axis): first index on ties */
                R best = q[0];
                for (int a = 1; a < 3; ++a) {
                    if (q[a] > best) {
                        best = q[a];
                        axis = a;
                    }
                }
                gg[0] = gg[1] = gg[2] = 0.0f;
                gg[axis] = sgn[axis];
            }
            for (int a = 0; a < 3; ++a) g[a] = pr->interior ? -gg[a] : gg[a];
            return;
        }
        default: {
            R gg[3];
            R q[3] = {p[0], p[1], p[2]};
            for (int a = 0; a < 3; ++a) {
                q[a] = p[a] + step;
                const R hi = cone_distance(pr, q);
                q[a] = p[a] - step;
                const R lo = cone_distance(pr, q);
                q[a] = p[a];
                gg[a] = (hi - lo) / (2.0f * step);
            }
            const R len = norm3(gg);
            if (len <= 0.0f) {
                g[0] = 0.0f;
                g[1] = 1.0f;
                g[2] = 0.0f;
                return;
            }
            g[0] = gg[0] / len;
            g[1] = gg[1] / len;
            g[2] = gg[2] / len;
            return;
        }
    }
}

/* sceneDistance (sdf.hpp:202-223); the scene is non-empty. */
static R scene_distance(const scene_t* sc, const R* p, R* grad) {
    R best = INFINITY;
    int bestIdx = 0;
    for (int k = 0; k < sc->n; ++k) {
        const R d = prim_distance(&sc->prims[k], p);
        if (d < best) {
            best = d;
            bestIdx = k;
        }
    }
    prim_gradient(&sc->prims[bestIdx], p, sc->step, grad);
    return best;
}

int32_t orc_scene_distance(const apbf_sdf_primitive* prims, int32_t n_prims, float gradient_step,
                           const float p[3], float* phi, float grad[3], apbf_error* err) {
    clear_err(err);
    scene_t sc;
    int32_t rc = scene_init(&sc, prims, n_prims, gradient_step, err);
    if (rc) return rc;
    if (sc.n == 0)
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "scene distance query on empty scene");
    *phi = scene_distance(&sc, p, grad);
    free(sc.prims);
    return APBF_OK;
}

/* findContacts(...).size() (sdf.hpp:226-250). */
static int64_t count_contacts(const scene_t* sc, int n, const R* pos, R r) {
    if (sc->n == 0) return 0;
    int64_t c = 0;
    for (int i = 0; i < n; ++i) {
        R g[3];
        if (scene_distance(sc, pos + 3 * i, g) < r) ++c;
    }
    return c;
}

int32_t orc_count_contacts(int32_t n, const float* positions, const apbf_sdf_primitive* prims,
                           int32_t n_prims, float gradient_step, float radius, int64_t* count_out,
                           apbf_error* err) {
    clear_err(err);
    scene_t sc;
    int32_t rc = scene_init(&sc, prims, n_prims, gradient_step, err);
    if (rc) return rc;
    *count_out = count_contacts(&sc, n, positions, radius);
    free(sc.prims);
    return APBF_OK;
}

/* ------------------------------------------------------------ uniform grid */

typedef struct {
    R h, h2;
    R origin[3];
    int32_t dims[3];
    int64_t cells;
    int32_t* cell_start; /* cells + 1 */
    int32_t* perm;       /* n */
    R* points;           /* 3n, sorted copy */
    int n;
} grid_t;

static void grid_free(grid_t* g) {
    free(g->cell_start);
    free(g->perm);
    free(g->points);
    memset(g, 0, sizeof *g);
}

/* UniformGrid::cellCoord (uniform_grid.hpp:117-125). */
static void cell_coord(const grid_t* g, const R* p, int* c) {
    for (int a = 0; a < 3; ++a) {
        const int v = (int)floorf((p[a] - g->origin[a]) / g->h);
        c[a] = mini_std(maxi_std(v, 0), g->dims[a] - 1);
    }
}

/* UniformGrid::linearCell (uniform_grid.hpp:216-218). */
static int linear_cell(const grid_t* g, const int* c) {
    return (int)(((int64_t)c[2] * g->dims[1] + c[1]) * g->dims[0] + c[0]);
}

/* UniformGrid::build (uniform_grid.hpp:42-98). */
static int32_t grid_build(grid_t* g, int n, const R* pos, R h, R pad, apbf_error* err) {
    grid_free(g);
    if (!(h > 0.0f))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "grid cell size must be positive");
    if (pad < 0.0f)
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "grid padding must be non-negative");
    g->h = h;
    g->h2 = h * h;
    g->n = n;
    if (n == 0) {
        g->dims[0] = g->dims[1] = g->dims[2] = 1;
        g->cells = 1;
        g->cell_start = (int32_t*)calloc(2, sizeof(int32_t));
        return APBF_OK;
    }
    for (int i = 0; i < n; ++i)
        if (!all_finite3(pos + 3 * i)) return numerical(err, "grid build", i, "non-finite position");
    R lo[3], hi[3];
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pos[a];
    for (int i = 1; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            const R v = pos[3 * i + a];
            if (v < lo[a]) lo[a] = v;
            if (v > hi[a]) hi[a] = v;
        }
    }
    R top[3];
    for (int a = 0; a < 3; ++a) {
        g->origin[a] = lo[a] - pad;
        top[a] = hi[a] + pad;
    }
    int64_t cells = 1;
    for (int a = 0; a < 3; ++a) {
        const R extent = top[a] - g->origin[a];
        g->dims[a] = maxi_std(1, (int)floorf(extent / h) + 1);
        cells *= g->dims[a];
        if (cells > K_MAX_CELLS)
            return set_err(err, APBF_ERR_RUNTIME, "", -1,
                           "grid cell count exceeds limit; domain blew up");
    }
    g->cells = cells;
    int32_t* cellOf = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    g->cell_start = (int32_t*)calloc((size_t)cells + 1, sizeof(int32_t));
    for (int i = 0; i < n; ++i) {
        int c[3];
        cell_coord(g, pos + 3 * i, c);
        const int id = linear_cell(g, c);
        cellOf[i] = id;
        ++g->cell_start[id + 1];
    }
    for (int64_t c = 1; c <= cells; ++c) g->cell_start[c] += g->cell_start[c - 1];
    g->perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* cursor = (int32_t*)malloc(sizeof(int32_t) * (size_t)cells);
    memcpy(cursor, g->cell_start, sizeof(int32_t) * (size_t)cells);
    for (int i = 0; i < n; ++i) g->perm[cursor[cellOf[i]]++] = i;
    free(cursor);
    free(cellOf);
    g->points = (R*)malloc(sizeof(R) * 3 * (size_t)(n > 0 ? n : 0));
    for (int k = 0; k < n; ++k)
        for (int a = 0; a < 3; ++a) g->points[3 * k + a] = pos[3 * g->perm[k] + a];
    return APBF_OK;
}

/* UniformGrid::forEachNeighbor (uniform_grid.hpp:135-158).  Calls fn for
 * each stored slot strictly within h of p, ascending. */
typedef void (*nbr_fn)(void* ctx, int k, R r2);
static void for_each_neighbor(const grid_t* g, const R* p, nbr_fn fn, void* ctx) {
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        const int c = (int)floorf((p[a] - g->origin[a]) / g->h);
        lo[a] = maxi_std(c - 1, 0);
        hi[a] = mini_std(c + 1, g->dims[a] - 1);
        if (lo[a] > hi[a]) return;
    }
    const R q[3] = {p[0], p[1], p[2]};
    for (int cz = lo[2]; cz <= hi[2]; ++cz) {
        for (int cy = lo[1]; cy <= hi[1]; ++cy) {
            const int64_t rowBase = ((int64_t)cz * g->dims[1] + cy) * g->dims[0];
            const int b = g->cell_start[rowBase + lo[0]];
            const int e = g->cell_start[rowBase + hi[0] + 1];
            for (int k = b; k < e; ++k) {
                const R d[3] = {q[0] - g->points[3 * k], q[1] - g->points[3 * k + 1],
                                q[2] - g->points[3 * k + 2]};
                const R r2 = sqn3(d);
                if (r2 < g->h2) fn(ctx, k, r2);
            }
        }
    }
}

typedef struct {
    int32_t* out;
    int64_t w;
} fill_ctx;
static void count_cb(void* ctx, int k, R r2) {
    (void)k;
    (void)r2;
    ++((fill_ctx*)ctx)->w;
}
static void fill_cb(void* ctx, int k, R r2) {
    (void)r2;
    fill_ctx* f = (fill_ctx*)ctx;
    f->out[f->w++] = k;
}

typedef struct {
    int32_t* offsets; /* n + 1 */
    int32_t* indices;
    int64_t total;
} lists_t;

static void lists_free(lists_t* l) {
    free(l->offsets);
    free(l->indices);
    memset(l, 0, sizeof *l);
}

/* UniformGrid::buildNeighborLists (uniform_grid.hpp:179-213): ascending,
 * self included, built from the stored (build-time) points. */
static int32_t build_lists(const grid_t* g, lists_t* l, apbf_error* err) {
    lists_free(l);
    const int n = g->n;
    l->offsets = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    int64_t total = 0;
    for (int i = 0; i < n; ++i) {
        fill_ctx c = {NULL, 0};
        for_each_neighbor(g, g->points + 3 * i, count_cb, &c);
        total += c.w;
        if (total > 2147483647LL)
            return set_err(err, APBF_ERR_RUNTIME, "", -1, "neighbor list overflow");
        l->offsets[i + 1] = (int32_t)total;
    }
    l->total = total;
    l->indices = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total > 0 ? total : 1));
    for (int i = 0; i < n; ++i) {
        fill_ctx c = {l->indices, l->offsets[i]};
        for_each_neighbor(g, g->points + 3 * i, fill_cb, &c);
    }
    return APBF_OK;
}

int32_t orc_grid_build(int32_t n, const float* positions, float h, float padding, int32_t* perm,
                       float* origin, int32_t* dims, int32_t* cell_start,
                       int64_t cell_start_capacity, int64_t* cells_out, apbf_error* err) {
    clear_err(err);
    grid_t g;
    memset(&g, 0, sizeof g);
    int32_t rc = grid_build(&g, n, positions, h, padding, err);
    if (rc) {
        grid_free(&g);
        return rc;
    }
    if (perm && n > 0) memcpy(perm, g.perm, sizeof(int32_t) * (size_t)n);
    if (origin) memcpy(origin, g.origin, sizeof g.origin);
    if (dims) memcpy(dims, g.dims, sizeof g.dims);
    if (cells_out) *cells_out = g.cells;
    if (cell_start) {
        if (cell_start_capacity < g.cells + 1) {
            grid_free(&g);
            return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "cell_start capacity too small");
        }
        memcpy(cell_start, g.cell_start, sizeof(int32_t) * (size_t)(g.cells + 1));
    }
    grid_free(&g);
    return APBF_OK;
}

int32_t orc_neighbor_lists(int32_t n, const float* positions, float h, float padding,
                           int32_t* offsets, int32_t* indices, int64_t indices_capacity,
                           int64_t* total_out, apbf_error* err) {
    clear_err(err);
    grid_t g;
    memset(&g, 0, sizeof g);
    lists_t l;
    memset(&l, 0, sizeof l);
    int32_t rc = grid_build(&g, n, positions, h, padding, err);
    if (!rc) rc = build_lists(&g, &l, err);
    if (!rc) {
        if (total_out) *total_out = l.total;
        if (offsets) memcpy(offsets, l.offsets, sizeof(int32_t) * ((size_t)n + 1));
        if (indices) {
            if (indices_capacity < l.total)
                rc = set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "indices capacity too small");
            else
                memcpy(indices, l.indices, sizeof(int32_t) * (size_t)l.total);
        }
    }
    lists_free(&l);
    grid_free(&g);
    return rc;
}

/* ------------------------------------------------------- solver passes */

/* computeDensity (solver.hpp:82-93). */
float orc_compute_density(int32_t i, const int32_t* offsets, const int32_t* indices,
                          const float* masses, const float* positions, float h) {
    const R* xi = positions + 3 * i;
    R rho = 0.0f;
    for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
        const int j = indices[e];
        const R d[3] = {xi[0] - positions[3 * j], xi[1] - positions[3 * j + 1],
                        xi[2] - positions[3 * j + 2]};
        rho += masses[j] * orc_density_kernel_r2(sqn3(d), h);
    }
    return rho;
}

/* computeLambda (solver.hpp:98-120). */
float orc_compute_lambda(int32_t i, const int32_t* offsets, const int32_t* indices,
                         const float* xs, const float* mass, const float* inv_mass,
                         const apbf_solver_config* cfg) {
    const R invRho0 = 1.0f / cfg->rest_density;
    const R* xi = xs + 3 * i;
    R rho = 0.0f;
    R gradI[3] = {0.0f, 0.0f, 0.0f};
    R denomJ = 0.0f;
    for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
        const int j = indices[e];
        const R rij[3] = {xi[0] - xs[3 * j], xi[1] - xs[3 * j + 1], xi[2] - xs[3 * j + 2]};
        rho += mass[j] * orc_density_kernel_r2(sqn3(rij), cfg->h);
        if (j != i) {
            R g[3];
            orc_gradient_kernel(rij, cfg->h, g);
            gradI[0] += g[0];
            gradI[1] += g[1];
            gradI[2] += g[2];
            denomJ += inv_mass[j] * sqn3(g);
        }
    }
    const R c = rho * invRho0 - 1.0f;
    const R sg[3] = {invRho0 * gradI[0], invRho0 * gradI[1], invRho0 * gradI[2]};
    const R denom = inv_mass[i] * sqn3(sg) + invRho0 * invRho0 * denomJ + cfg->epsilon;
    return -c / denom;
}

/* computeDeltaP (solver.hpp:125-141). */
void orc_compute_deltap(int32_t i, const int32_t* offsets, const int32_t* indices,
                        const float* xs, const float* inv_mass, const float* lambda,
                        const int32_t* level, const apbf_solver_config* cfg, int32_t iteration,
                        float out[3]) {
    const R* xi = xs + 3 * i;
    const R lamI = lambda[i];
    R sum[3] = {0.0f, 0.0f, 0.0f};
    for (int e = offsets[i]; e < offsets[i + 1]; ++e) {
        const int j = indices[e];
        if (j == i) continue;
        R lamJ = lambda[j];
        if (cfg->inactive_lambda_zero && iteration > 0 && !(level[j] >= iteration)) lamJ = 0.0f;
        const R rij[3] = {xi[0] - xs[3 * j], xi[1] - xs[3 * j + 1], xi[2] - xs[3 * j + 2]};
        R g[3];
        orc_gradient_kernel(rij, cfg->h, g);
        const R s = lamI + lamJ;
        sum[0] += s * g[0];
        sum[1] += s * g[1];
        sum[2] += s * g[2];
    }
    const R k = inv_mass[i] / cfg->rest_density;
    out[0] = k * sum[0];
    out[1] = k * sum[1];
    out[2] = k * sum[2];
}

/* allDensities (solver.hpp:145-162): rho in original index order. */
static int32_t all_densities(int n, const R* pos, const R* masses, R h, R* rho, apbf_error* err) {
    if (n == 0) return APBF_OK;
    grid_t g;
    memset(&g, 0, sizeof g);
    lists_t l;
    memset(&l, 0, sizeof l);
    int32_t rc = grid_build(&g, n, pos, h, h, err);
    if (!rc) rc = build_lists(&g, &l, err);
    if (!rc) {
        R* sortedMass = (R*)malloc(sizeof(R) * (size_t)n);
        for (int k = 0; k < n; ++k) sortedMass[k] = masses[g.perm[k]];
        for (int k = 0; k < n; ++k)
            rho[g.perm[k]] = orc_compute_density(k, l.offsets, l.indices, sortedMass, g.points, h);
        free(sortedMass);
    }
    lists_free(&l);
    grid_free(&g);
    return rc;
}

int32_t orc_all_densities(int32_t n, const float* positions, const float* masses, float h,
                          float* rho_out, apbf_error* err) {
    clear_err(err);
    return all_densities(n, positions, masses, h, rho_out, err);
}

/* ------------------------------------------------------- camera / splat */

typedef struct {
    R eye[3], forward[3], right[3], trueUp[3];
    R tanX, tanY;
    int width, height;
    R nearClip;
} camframe_t;

/* Camera::validate (depth_splat.hpp:29-42). */
static int32_t camera_validate(const apbf_camera* cam, apbf_error* err) {
    if (cam->width <= 0 || cam->height <= 0)
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                       "camera resolution must be positive in both axes");
    const R d[3] = {cam->look_at[0] - cam->eye[0], cam->look_at[1] - cam->eye[1],
                    cam->look_at[2] - cam->eye[2]};
    if (!(sqn3(d) > 0.0f))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "camera look-at must differ from eye");
    if (!(cam->vertical_fov > 0.0f) || !(cam->vertical_fov < PI_F))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "vertical fov must lie in (0, pi)");
    if (!(cam->near_clip > 0.0f))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "near clip must be positive");
    return APBF_OK;
}

/* CameraFrame::CameraFrame (depth_splat.hpp:55-71). */
static int32_t camframe_init(camframe_t* f, const apbf_camera* cam, apbf_error* err) {
    int32_t rc = camera_validate(cam, err);
    if (rc) return rc;
    R d[3] = {cam->look_at[0] - cam->eye[0], cam->look_at[1] - cam->eye[1],
              cam->look_at[2] - cam->eye[2]};
    const R z = sqn3(d); /* normalized(): v / sqrt(sqn) when sqn > 0 */
    if (z > 0.0f) {
        const R s = sqrtf(z);
        d[0] /= s;
        d[1] /= s;
        d[2] /= s;
    }
    memcpy(f->eye, cam->eye, sizeof f->eye);
    memcpy(f->forward, d, sizeof d);
    cross3(f->forward, cam->up, f->right);
    const R len = norm3(f->right);
    if (!(len > 1e-12f))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                       "camera up is parallel to the view direction");
    f->right[0] /= len;
    f->right[1] /= len;
    f->right[2] /= len;
    cross3(f->right, f->forward, f->trueUp);
    f->tanY = tanf(cam->vertical_fov / 2.0f);
    f->tanX = f->tanY * (R)cam->width / (R)cam->height;
    f->width = cam->width;
    f->height = cam->height;
    f->nearClip = cam->near_clip;
    return APBF_OK;
}

typedef struct {
    R u, v, zForward, distance;
    int inFront, onScreen;
} projection_t;

/* CameraFrame::project (depth_splat.hpp:81-96). */
static projection_t project(const camframe_t* f, const R* p) {
    projection_t pr = {0, 0, 0, 0, 0, 0};
    const R rel[3] = {p[0] - f->eye[0], p[1] - f->eye[1], p[2] - f->eye[2]};
    pr.zForward = dot3(rel, f->forward);
    pr.distance = norm3(rel);
    if (!(pr.zForward > f->nearClip)) return pr;
    pr.inFront = 1;
    const R sx = dot3(rel, f->right) / (pr.zForward * f->tanX);
    const R sy = dot3(rel, f->trueUp) / (pr.zForward * f->tanY);
    pr.u = (sx + 1.0f) / 2.0f * (R)f->width;
    pr.v = (1.0f - sy) / 2.0f * (R)f->height;
    pr.onScreen = pr.u >= 0.0f && pr.u < (R)f->width && pr.v >= 0.0f && pr.v < (R)f->height;
    return pr;
}

/* detail::splatSphere (depth_splat.hpp:138-194) with min-compositing into
 * depth (depth_splat.hpp:215-218). */
static void splat_sphere(const camframe_t* f, const R* center, R r, R* depth) {
    const R rel[3] = {center[0] - f->eye[0], center[1] - f->eye[1], center[2] - f->eye[2]};
    const R z = dot3(rel, f->forward);
    if (!(z > f->nearClip)) return;
    const R q = sqn3(rel);
    const R r2 = r * r;
    int x0 = 0, x1 = f->width - 1, y0 = 0, y1 = f->height - 1;
    if (q > r2) {
        const R cx = dot3(rel, f->right) / z;
        const R cy = dot3(rel, f->trueUp) / z;
        const R tana = r / sqrtf(q - r2);
        const R rho = sqrtf(cx * cx + cy * cy);
        if (tana * rho < 1.0f) {
            const R u = (cx / f->tanX + 1.0f) / 2.0f * (R)f->width;
            const R v = (1.0f - cy / f->tanY) / 2.0f * (R)f->height;
            const R ext = tana * (1.0f + rho * rho) / (1.0f - tana * rho);
            const R eu = ext / f->tanX * (R)f->width / 2.0f;
            const R ev = ext / f->tanY * (R)f->height / 2.0f;
            const R w = (R)f->width, h = (R)f->height;
            x0 = maxi_std(0, (int)floorf(clampf_std(u - eu, 0.0f, w)) - 1);
            x1 = mini_std(f->width - 1, (int)ceilf(clampf_std(u + eu, -1.0f, w)) + 1);
            y0 = maxi_std(0, (int)floorf(clampf_std(v - ev, 0.0f, h)) - 1);
            y1 = mini_std(f->height - 1, (int)ceilf(clampf_std(v + ev, -1.0f, h)) + 1);
        }
    }
    for (int iy = y0; iy <= y1; ++iy) {
        const R ry = (1.0f - ((R)iy + 0.5f) / (R)f->height * 2.0f) * f->tanY;
        const R rowBase[3] = {f->forward[0] + ry * f->trueUp[0], f->forward[1] + ry * f->trueUp[1],
                              f->forward[2] + ry * f->trueUp[2]};
        for (int ix = x0; ix <= x1; ++ix) {
            const R rx = (((R)ix + 0.5f) / (R)f->width * 2.0f - 1.0f) * f->tanX;
            const R d[3] = {rowBase[0] + rx * f->right[0], rowBase[1] + rx * f->right[1],
                            rowBase[2] + rx * f->right[2]};
            const R a = sqn3(d);
            const R b = dot3(d, rel);
            const R disc = b * b - a * (q - r2);
            if (disc < 0.0f) continue;
            const R t = (b - sqrtf(disc)) / sqrtf(a);
            if (t > f->nearClip) {
                R* cell = depth + (size_t)iy * (size_t)f->width + ix;
                if (t < *cell) *cell = t;
            }
        }
    }
}

/* splat (depth_splat.hpp:201-228). */
static int32_t splat(int n, const R* pos, R r, const apbf_camera* cam, R* depth, apbf_error* err) {
    if (!(r > 0.0f))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "splat radius must be positive");
    camframe_t f;
    int32_t rc = camframe_init(&f, cam, err);
    if (rc) return rc;
    const size_t px = (size_t)cam->width * (size_t)cam->height;
    for (size_t k = 0; k < px; ++k) depth[k] = INFINITY;
    for (int i = 0; i < n; ++i) splat_sphere(&f, pos + 3 * i, r, depth);
    return APBF_OK;
}

int32_t orc_splat(int32_t n, const float* positions, float radius, const apbf_camera* cam,
                  float* depth_out, apbf_error* err) {
    clear_err(err);
    return splat(n, positions, radius, cam, depth_out, err);
}

/* ------------------------------------------------------------------ LOD */

/* mapDistanceToLevel (lod.hpp:33-40). */
int32_t orc_map_distance_to_level(float d, float dMin, float dMax, int32_t nMin, int32_t nMax) {
    if (!(dMax > dMin)) return nMax;
    R t = (d - dMin) / (dMax - dMin);
    t = clampf_std(t, 0.0f, 1.0f);
    const int level = (int)roundf((R)nMax + t * (R)(nMin - nMax));
    return level < nMin ? nMin : (nMax < level ? nMax : level);
}

static int cmp_float(const void* a, const void* b) {
    const R x = *(const R*)a, y = *(const R*)b;
    return (x < y) ? -1 : (y < x) ? 1 : 0;
}

/* sortedPercentile (lod.hpp:49-60). */
static R sorted_percentile(const R* v, size_t n, R p) {
    const R pos = p / 100.0f * (R)(n - 1);
    const size_t lo = (size_t)floorf(pos);
    const size_t hi = (lo + 1 < n - 1) ? lo + 1 : n - 1;
    const R frac = pos - (R)lo;
    return v[lo] * (1.0f - frac) + v[hi] * frac;
}

float orc_percentile(const float* values, int32_t n, float p) {
    if (n <= 0) return NAN;
    R* s = (R*)malloc(sizeof(R) * (size_t)n);
    memcpy(s, values, sizeof(R) * (size_t)n);
    qsort(s, (size_t)n, sizeof(R), cmp_float);
    const R r = sorted_percentile(s, (size_t)n, p);
    free(s);
    return r;
}

/* resolveAutoRange (lod.hpp:71-78). */
static int resolve_auto_range(const R* sample, size_t n, R* dMin, R* dMax) {
    R* s = (R*)malloc(sizeof(R) * n);
    memcpy(s, sample, sizeof(R) * n);
    qsort(s, n, sizeof(R), cmp_float);
    *dMin = sorted_percentile(s, n, 5.0f);
    *dMax = sorted_percentile(s, n, 95.0f);
    free(s);
    return *dMax > *dMin;
}

static int32_t lod_validate(const apbf_lod_config* lod, apbf_error* err) {
    if (!lod->auto_range && !(lod->d_min < lod->d_max))
        return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                       "lod distance range requires d_min < d_max");
    return APBF_OK;
}

/* lodDtc (lod.hpp:83-104). */
static int32_t lod_dtc(int n, const R* pos, const apbf_camera* cam, const apbf_lod_config* lod,
                       int32_t* levels, apbf_error* err) {
    int32_t rc = lod_validate(lod, err);
    if (rc || n <= 0) return rc;
    R* dist = (R*)calloc((size_t)n, sizeof(R));
    for (int i = 0; i < n; ++i) {
        const R d[3] = {pos[3 * i] - cam->eye[0], pos[3 * i + 1] - cam->eye[1],
                        pos[3 * i + 2] - cam->eye[2]};
        dist[i] = norm3(d);
    }
    R dMin = lod->d_min, dMax = lod->d_max;
    if (lod->auto_range && !resolve_auto_range(dist, (size_t)n, &dMin, &dMax)) {
        for (int i = 0; i < n; ++i) levels[i] = lod->n_max;
        free(dist);
        return APBF_OK;
    }
    for (int i = 0; i < n; ++i)
        levels[i] = orc_map_distance_to_level(dist[i], dMin, dMax, lod->n_min, lod->n_max);
    free(dist);
    return APBF_OK;
}

/* lodDtvs (lod.hpp:109-156). */
static int32_t lod_dtvs(int n, const R* pos, const apbf_camera* cam, const apbf_lod_config* lod,
                        R r, int32_t* levels, apbf_error* err) {
    int32_t rc = lod_validate(lod, err);
    if (rc || n == 0) return rc;
    R* depth = (R*)malloc(sizeof(R) * (size_t)(cam->width > 0 ? cam->width : 1) *
                          (size_t)(cam->height > 0 ? cam->height : 1));
    rc = splat(n, pos, r, cam, depth, err);
    if (rc) {
        free(depth);
        return rc;
    }
    camframe_t f;
    camframe_init(&f, cam, err);
    R* gap = (R*)calloc((size_t)n, sizeof(R));
    char* visible = (char*)calloc((size_t)n, 1);
    for (int i = 0; i < n; ++i) {
        const projection_t pr = project(&f, pos + 3 * i);
        if (!pr.inFront || !pr.onScreen) continue;
        const int px = mini_std((int)pr.u, cam->width - 1);
        const int py = mini_std((int)pr.v, cam->height - 1);
        R d = pr.distance - depth[(size_t)py * (size_t)cam->width + px];
        if (d < r) d = 0.0f;
        gap[i] = maxf_std(d, 0.0f);
        visible[i] = 1;
    }
    R dMin = lod->d_min, dMax = lod->d_max;
    int spread = 1;
    if (lod->auto_range) {
        R* sample = (R*)malloc(sizeof(R) * (size_t)(n > 0 ? n : 0));
        size_t m = 0;
        for (int i = 0; i < n; ++i)
            if (visible[i]) sample[m++] = gap[i];
        if (m == 0) {
            for (int i = 0; i < n; ++i) levels[i] = lod->n_min;
            free(sample);
            free(gap);
            free(visible);
            free(depth);
            return APBF_OK;
        }
        spread = resolve_auto_range(sample, m, &dMin, &dMax);
        free(sample);
    }
    for (int i = 0; i < n; ++i) {
        if (!visible[i])
            levels[i] = lod->n_min;
        else if (!spread)
            levels[i] = lod->n_max;
        else
            levels[i] = orc_map_distance_to_level(gap[i], dMin, dMax, lod->n_min, lod->n_max);
    }
    free(gap);
    free(visible);
    free(depth);
    return APBF_OK;
}

int32_t orc_lod_dtc(int32_t n, const float* positions, const apbf_camera* cam,
                    const apbf_lod_config* lod, int32_t* levels_out, apbf_error* err) {
    clear_err(err);
    return lod_dtc(n, positions, cam, lod, levels_out, err);
}

int32_t orc_lod_dtvs(int32_t n, const float* positions, const apbf_camera* cam,
                     const apbf_lod_config* lod, float radius, int32_t* levels_out,
                     apbf_error* err) {
    clear_err(err);
    return lod_dtvs(n, positions, cam, lod, radius, levels_out, err);
}

/* --------------------------------------------------------------- solver */

struct orc_solver {
    apbf_solver_config cfg;
    scene_t scene;
    int n;
    R *x, *xs, *v, *mass, *invMass, *lambda, *deltaP;
    int32_t* level;
    grid_t grid;
    lists_t nl;
    int32_t* order;
    int64_t* activeCount; /* nMax + 2 */
    apbf_iteration_observer observer;
    void* observer_user;
    int metrics;
};

/* SolverConfig derived values (solver.hpp:44-51). */
static R dt_substep(const apbf_solver_config* c) { return c->dt_frame / (R)c->substeps; }
static int stab_threshold(const apbf_solver_config* c) {
    return c->stab_threshold > 0 ? c->stab_threshold : c->n_max;
}
static R particle_radius(const apbf_solver_config* c) {
    return c->particle_radius > 0.0f ? c->particle_radius : c->h / 4.0f;
}
static R velocity_cap(const apbf_solver_config* c) {
    return c->velocity_cap > 0.0f ? c->velocity_cap : c->h / dt_substep(c);
}

/* IterationRange ctor + SolverConfig::validate (particle_state.hpp:22-26,
 * solver.hpp:53-66). */
static int32_t validate_config(const apbf_solver_config* c, apbf_error* err) {
#define BAD(msg) return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, msg)
    if (c->n_min < 1 || c->n_max < c->n_min) BAD("iteration range requires 1 <= n_min <= n_max");
    if (!(c->dt_frame > 0.0f)) BAD("dt_frame must be positive");
    if (c->substeps < 1) BAD("substeps must be at least 1");
    if (!(c->rest_density > 0.0f)) BAD("rest density must be positive");
    if (!(c->h > 0.0f)) BAD("smoothing length must be positive");
    if (c->epsilon < 0.0f) BAD("epsilon must be non-negative");
    if (c->stab_iterations < 0) BAD("stab iterations must be non-negative");
    if (c->stab_threshold != 0 && (c->stab_threshold < 1 || c->stab_threshold > c->n_max))
        BAD("stab threshold must lie in [1, n_max]");
    if (c->particle_radius < 0.0f) BAD("particle radius must be non-negative");
    if (c->velocity_cap < 0.0f) BAD("velocity cap must be non-negative");
    if (!all_finite3(c->gravity)) BAD("gravity must be finite");
    if (c->mode != APBF_MODE_PBF && c->mode != APBF_MODE_APBF) BAD("unknown solver mode");
#undef BAD
    return APBF_OK;
}

orc_solver* orc_solver_create(const apbf_solver_config* cfg, const apbf_sdf_primitive* prims,
                              int32_t n_prims, float gradient_step, apbf_error* err) {
    clear_err(err);
    if (validate_config(cfg, err)) return NULL;
    orc_solver* s = (orc_solver*)calloc(1, sizeof(orc_solver));
    s->cfg = *cfg;
    if (scene_init(&s->scene, prims, n_prims, gradient_step, err)) {
        free(s);
        return NULL;
    }
    s->metrics = 1;
    return s;
}

static void free_state(orc_solver* s) {
    free(s->x);
    free(s->xs);
    free(s->v);
    free(s->mass);
    free(s->invMass);
    free(s->lambda);
    free(s->deltaP);
    free(s->level);
    free(s->order);
    s->x = s->xs = s->v = s->mass = s->invMass = s->lambda = s->deltaP = NULL;
    s->level = s->order = NULL;
}

void orc_solver_destroy(orc_solver* s) {
    if (!s) return;
    free_state(s);
    grid_free(&s->grid);
    lists_free(&s->nl);
    free(s->activeCount);
    free(s->scene.prims);
    free(s);
}

int32_t orc_set_state(orc_solver* s, int32_t n, const float* x, const float* xs, const float* v,
                      const float* mass, const float* invMass, const float* lambda,
                      const int32_t* level, apbf_error* err) {
    clear_err(err);
    if (n < 0) return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1, "negative particle count");
    free_state(s);
    s->n = n;
    const size_t n3 = sizeof(R) * 3 * (size_t)(n > 0 ? n : 1);
    const size_t n1 = sizeof(R) * (size_t)(n > 0 ? n : 1);
    s->x = (R*)malloc(n3);
    s->xs = (R*)malloc(n3);
    s->v = (R*)malloc(n3);
    s->deltaP = (R*)calloc(1, n3);
    s->mass = (R*)malloc(n1);
    s->invMass = (R*)malloc(n1);
    s->lambda = (R*)malloc(n1);
    s->level = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    s->order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (n > 0) {
        memcpy(s->x, x, n3);
        memcpy(s->xs, xs, n3);
        memcpy(s->v, v, n3);
        memcpy(s->mass, mass, n1);
        memcpy(s->invMass, invMass, n1);
        memcpy(s->lambda, lambda, n1);
        memcpy(s->level, level, sizeof(int32_t) * (size_t)n);
    }
    return APBF_OK;
}

int32_t orc_get_state(const orc_solver* s, float* x, float* xs, float* v, float* mass,
                      float* invMass, float* lambda, int32_t* level) {
    const size_t n3 = sizeof(R) * 3 * (size_t)s->n, n1 = sizeof(R) * (size_t)s->n;
    if (s->n == 0) return APBF_OK;
    if (x) memcpy(x, s->x, n3);
    if (xs) memcpy(xs, s->xs, n3);
    if (v) memcpy(v, s->v, n3);
    if (mass) memcpy(mass, s->mass, n1);
    if (invMass) memcpy(invMass, s->invMass, n1);
    if (lambda) memcpy(lambda, s->lambda, n1);
    if (level) memcpy(level, s->level, sizeof(int32_t) * (size_t)s->n);
    return APBF_OK;
}

void orc_set_iteration_observer(orc_solver* s, apbf_iteration_observer cb, void* user) {
    s->observer = cb;
    s->observer_user = user;
}

void orc_set_frame_metrics(orc_solver* s, int32_t enabled) { s->metrics = enabled; }

int32_t orc_last_permutation(const orc_solver* s, int32_t* perm) {
    if (s->grid.n > 0) memcpy(perm, s->grid.perm, sizeof(int32_t) * (size_t)s->grid.n);
    return s->grid.n;
}

/* ParticleSet::applyPermutation (particle_state.hpp:74-98). */
static void apply_permutation(orc_solver* s, const int32_t* perm) {
    const int n = s->n;
    R* t3 = (R*)malloc(sizeof(R) * 3 * (size_t)n);
    R* t1 = (R*)malloc(sizeof(R) * (size_t)n);
    int32_t* ti = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    R** f3[3] = {&s->x, &s->xs, &s->v};
    for (int f = 0; f < 3; ++f) {
        R* a = *f3[f];
        for (int k = 0; k < n; ++k)
            for (int c = 0; c < 3; ++c) t3[3 * k + c] = a[3 * perm[k] + c];
        *f3[f] = t3;
        t3 = a;
    }
    R** f1[3] = {&s->mass, &s->invMass, &s->lambda};
    for (int f = 0; f < 3; ++f) {
        R* a = *f1[f];
        for (int k = 0; k < n; ++k) t1[k] = a[perm[k]];
        *f1[f] = t1;
        t1 = a;
    }
    for (int k = 0; k < n; ++k) ti[k] = s->level[perm[k]];
    free(s->level);
    s->level = ti;
    free(t3);
    free(t1);
}

/* detail::checkFiniteCols / checkFiniteVec (solver.hpp:184-202). */
static int first_nonfinite3(const R* a, int n) {
    for (int i = 0; i < n; ++i)
        if (!all_finite3(a + 3 * i)) return i;
    return -1;
}
static int first_nonfinite1(const R* a, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(a[i])) return i;
    return -1;
}

/* Solver::buildIterationOrder (solver.hpp:361-380). */
static void build_iteration_order(orc_solver* s) {
    const int n = s->n, top = s->cfg.n_max;
    int64_t* levelCount = (int64_t*)calloc((size_t)top + 2, sizeof(int64_t));
    for (int i = 0; i < n; ++i) ++levelCount[s->level[i]];
    free(s->activeCount);
    s->activeCount = (int64_t*)calloc((size_t)top + 2, sizeof(int64_t));
    for (int l = top; l >= 1; --l) s->activeCount[l] = s->activeCount[l + 1] + levelCount[l];
    int64_t* bucketStart = (int64_t*)calloc((size_t)top + 2, sizeof(int64_t));
    for (int l = top - 1; l >= 1; --l) bucketStart[l] = bucketStart[l + 1] + levelCount[l + 1];
    for (int i = 0; i < n; ++i) s->order[bucketStart[s->level[i]]++] = i;
    free(bucketStart);
    free(levelCount);
}

/* meanAbsConstraint (solver.hpp:166-180). */
static double mean_abs_constraint(const orc_solver* s) {
    const int n = s->n;
    if (n == 0) return 0.0;
    double sum = 0.0;
    for (int i = 0; i < n; ++i) {
        const R c = fabsf(orc_compute_density(i, s->nl.offsets, s->nl.indices, s->mass, s->xs,
                                              s->cfg.h) /
                              s->cfg.rest_density -
                          1.0f);
        sum += (double)c;
    }
    return sum / n;
}

static void push_residual(apbf_frame_stats* st, double r) {
    if (st->residuals && st->n_residuals < st->residuals_capacity)
        st->residuals[st->n_residuals] = r;
    st->n_residuals++;
}

/* Solver::substep (solver.hpp:282-357). */
static int32_t substep(orc_solver* s, int substepIndex, apbf_frame_stats* st, apbf_error* err) {
    const apbf_solver_config* cfg = &s->cfg;
    const R dt = dt_substep(cfg);
    const R radius = particle_radius(cfg);
    const int n = s->n;
    int bad;

    for (int i = 0; i < n; ++i) { /* :287-291 */
        R* v = s->v + 3 * i;
        for (int c = 0; c < 3; ++c) {
            v[c] += dt * cfg->gravity[c];
        }
        for (int c = 0; c < 3; ++c) s->xs[3 * i + c] = s->x[3 * i + c] + dt * v[c];
    }
    if ((bad = first_nonfinite3(s->xs, n)) >= 0)
        return numerical(err, "predict", bad, "non-finite predicted position");

    int32_t rc = grid_build(&s->grid, n, s->xs, cfg->h, cfg->h, err); /* :294 */
    if (rc) return rc;
    if (n > 0) apply_permutation(s, s->grid.perm);
    rc = build_lists(&s->grid, &s->nl, err); /* :295 */
    if (rc) return rc;
    if (s->scene.n > 0) st->contacts += count_contacts(&s->scene, n, s->xs, radius); /* :296-299 */

    /* finishedSet + prestabilize (:301-305, sdf.hpp:261-278) */
    const int S = stab_threshold(cfg);
    int anyFinished = 0;
    if (S > 1)
        for (int i = 0; i < n; ++i)
            if (!(s->level[i] >= S)) anyFinished = 1;
    if (s->scene.n > 0 && anyFinished && cfg->stab_iterations > 0) {
        for (int it = 0; it < cfg->stab_iterations; ++it) {
            for (int i = 0; i < n; ++i) {
                if (s->level[i] >= S) continue;
                R g[3];
                const R phi = scene_distance(&s->scene, s->xs + 3 * i, g);
                if (phi < radius) {
                    const R k = radius - phi;
                    for (int c = 0; c < 3; ++c) {
                        const R delta = k * g[c];
                        s->xs[3 * i + c] += delta;
                        s->x[3 * i + c] += delta;
                    }
                }
            }
        }
    }
    if (anyFinished && (bad = first_nonfinite3(s->xs, n)) >= 0)
        return numerical(err, "prestabilize", bad, "non-finite predicted position");

    build_iteration_order(s); /* :307 */

    for (int iter = 1; iter <= cfg->n_max; ++iter) { /* :310-345 */
        const int64_t active = s->activeCount[iter];
        if (active == 0) break;
        st->total_iterations += active;
        for (int64_t k = 0; k < active; ++k) {
            const int i = s->order[k];
            s->lambda[i] = orc_compute_lambda(i, s->nl.offsets, s->nl.indices, s->xs, s->mass,
                                              s->invMass, cfg);
        }
        if ((bad = first_nonfinite1(s->lambda, n)) >= 0)
            return numerical(err, "lambda", bad, "non-finite lambda");
        for (int64_t k = 0; k < active; ++k) {
            const int i = s->order[k];
            orc_compute_deltap(i, s->nl.offsets, s->nl.indices, s->xs, s->invMass, s->lambda,
                               s->level, cfg, iter, s->deltaP + 3 * i);
        }
        for (int64_t k = 0; k < active; ++k) {
            const int i = s->order[k];
            R* p = s->xs + 3 * i;
            for (int c = 0; c < 3; ++c) p[c] += s->deltaP[3 * i + c];
            if (s->scene.n > 0) {
                R g[3];
                const R phi = scene_distance(&s->scene, p, g);
                if (phi < radius) {
                    const R kk = radius - phi;
                    for (int c = 0; c < 3; ++c) p[c] += kk * g[c];
                }
            }
        }
        if ((bad = first_nonfinite3(s->xs, n)) >= 0)
            return numerical(err, "apply", bad, "non-finite predicted position");
        if (cfg->record_residuals) push_residual(st, mean_abs_constraint(s));
        if (s->observer) s->observer(s->observer_user, substepIndex, iter);
    }

    const R cap = velocity_cap(cfg); /* :347-356 */
    for (int i = 0; i < n; ++i) {
        R* v = s->v + 3 * i;
        for (int c = 0; c < 3; ++c) v[c] = (s->xs[3 * i + c] - s->x[3 * i + c]) / dt;
        const R speed = norm3(v);
        if (speed > cap) {
            const R f = cap / speed;
            for (int c = 0; c < 3; ++c) v[c] *= f;
        }
        for (int c = 0; c < 3; ++c) s->x[3 * i + c] = s->xs[3 * i + c];
    }
    if ((bad = first_nonfinite3(s->v, n)) >= 0)
        return numerical(err, "finalize", bad, "non-finite velocity");
    if ((bad = first_nonfinite3(s->x, n)) >= 0)
        return numerical(err, "finalize", bad, "non-finite position");
    return APBF_OK;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* Solver::runSubsteps (solver.hpp:260-280). */
static int32_t run_substeps(orc_solver* s, int frame, double t0, apbf_frame_stats* st,
                            apbf_error* err) {
    st->frame = frame;
    st->n_residuals = 0;
    st->total_iterations = 0;
    st->contacts = 0;
    st->avg_density_pct = st->min_density_pct = st->max_density_pct = 0.0;
    for (int k = 0; k < s->cfg.substeps; ++k) {
        int32_t rc = substep(s, k, st, err);
        if (rc) return rc;
    }
    st->wall_ms = now_ms() - t0;
    if (s->n > 0 && s->metrics) {
        R* rho = (R*)malloc(sizeof(R) * (size_t)s->n);
        int32_t rc = all_densities(s->n, s->x, s->mass, s->cfg.h, rho, err);
        if (rc) {
            free(rho);
            return rc;
        }
        double sum = 0.0;
        R lo = rho[0], hi = rho[0];
        for (int i = 0; i < s->n; ++i) {
            sum += (double)rho[i];
            if (rho[i] < lo) lo = rho[i];
            if (rho[i] > hi) hi = rho[i];
        }
        const double scale = 100.0 / (double)s->cfg.rest_density;
        st->avg_density_pct = sum / s->n * scale;
        st->min_density_pct = (double)lo * scale;
        st->max_density_pct = (double)hi * scale;
        free(rho);
    }
    return APBF_OK;
}

/* Solver::stepFrame + assignLevels (solver.hpp:228-233, 247-258). */
int32_t orc_step_frame(orc_solver* s, const apbf_camera* cam, const apbf_lod_config* lod,
                       int32_t frame_index, apbf_frame_stats* out, apbf_error* err) {
    clear_err(err);
    const double t0 = now_ms();
    if (s->cfg.mode == APBF_MODE_PBF) {
        for (int i = 0; i < s->n; ++i) s->level[i] = s->cfg.n_max;
    } else {
        apbf_lod_config lc = *lod;
        lc.n_min = s->cfg.n_min;
        lc.n_max = s->cfg.n_max;
        int32_t rc = lc.model == APBF_LOD_DTC
                         ? lod_dtc(s->n, s->x, cam, &lc, s->level, err)
                         : lod_dtvs(s->n, s->x, cam, &lc, particle_radius(&s->cfg), s->level, err);
        if (rc) return rc;
    }
    return run_substeps(s, frame_index, t0, out, err);
}

int32_t orc_step_frame_with_levels(orc_solver* s, int32_t frame_index, apbf_frame_stats* out,
                                   apbf_error* err) {
    clear_err(err);
    for (int i = 0; i < s->n; ++i) {
        if (!(s->cfg.n_min <= s->level[i] && s->level[i] <= s->cfg.n_max))
            return set_err(err, APBF_ERR_INVALID_ARGUMENT, "", -1,
                           "particle level outside configured iteration range");
    }
    return run_substeps(s, frame_index, now_ms(), out, err);
}

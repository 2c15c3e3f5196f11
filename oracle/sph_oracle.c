/*
 * sph_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference CPU density pass (package `sphlab`
 * under /root/reference/pkg/src/sphlab).  It is the checker the CUDA path is
 * compared against and the CPU baseline bench.py times.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
 * may load it.  The product library (paper_1612_06090_b200/) never links it.
 *
 * Pinning: the restatement is checked bit-for-bit (h, density, todo trace,
 * particle_perm, fixed-h counts) against golden vectors produced by running
 * the reference itself; see tests/golden/make_golden.py and
 * tests/test_oracle_golden.py.
 *
 * What is restated, with the reference lines it follows:
 *   - octree build: root cube + pad (octree.py:324-336), LIFO node stack,
 *     coincident-point guard, stable 8-way counting sort by the x-major
 *     octant code, child centres c +- half/2 (octree.py:36-176)
 *   - range query with the padded cube/sphere prune and the exact
 *     `d2 = (dx*dx + dy*dy) + dz*dz <= r*r` leaf test (octree.py:179-227)
 *   - K-nearest selection under the (d2, index) total order
 *     (selection.py:30-131; only the resulting ordered prefix matters)
 *   - the smoothing-length update (density.py:143-157, 215-246) and the
 *     density sum m_i W(0,h) + sum_{n<K} m_j W(r_n,h) in sorted order
 *     (density.py:160-171, 249-261), Wendland C6 (kernel.py:30-45)
 *   - the todo-list outer loop with ConvergenceError / Degenerate checks
 *     (density.py:365-391)
 * Compile with -ffp-contract=off: every fp64 operation must round exactly as
 * the reference's (numba/LLVM does not contract a*b+c into an FMA).
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WC6_NORM (1365.0 / (64.0 * 3.14159265358979323846))
#define NO_CHILD (-1)

/* status codes shared with include/sph_b200.h */
#define ST_OK 0
#define ST_NOT_CONVERGED 1
#define ST_DEGENERATE 2
#define ST_INVALID 3
#define ST_NOMEM 5

typedef struct {
    int64_t n_nodes, cap;
    double *c;       /* 3 * cap, centres, row-major like the reference */
    double *half;
    int64_t *child, *start, *end;
    int64_t *perm;   /* n */
    double pad;
    int64_t n;
    const double *x, *y, *z;
} otree;

static void otree_free(otree *t) {
    free(t->c); free(t->half); free(t->child); free(t->start); free(t->end);
    free(t->perm);
    memset(t, 0, sizeof(*t));
}

static int otree_grow(otree *t) {
    int64_t nc = t->cap * 2;
    double *c = realloc(t->c, sizeof(double) * 3 * nc);
    if (!c) return -1; t->c = c;
    double *h = realloc(t->half, sizeof(double) * nc);
    if (!h) return -1; t->half = h;
    int64_t *k = realloc(t->child, sizeof(int64_t) * nc);
    if (!k) return -1; t->child = k;
    int64_t *s = realloc(t->start, sizeof(int64_t) * nc);
    if (!s) return -1; t->start = s;
    int64_t *e = realloc(t->end, sizeof(int64_t) * nc);
    if (!e) return -1; t->end = e;
    t->cap = nc;
    return 0;
}

static inline int octant(double px, double py, double pz, double cx, double cy, double cz) {
    int o = 0;
    if (px >= cx) o += 4;
    if (py >= cy) o += 2;
    if (pz >= cz) o += 1;
    return o;
}

/* octree.py:306-348 + the _build_kernel it calls */
static int otree_build(otree *t, int64_t n, const double *x, const double *y,
                       const double *z, int64_t leaf_cap, int64_t max_depth) {
    memset(t, 0, sizeof(*t));
    t->n = n; t->x = x; t->y = y; t->z = z;
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(x[i]) || !isfinite(y[i]) || !isfinite(z[i])) return ST_INVALID;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, ctr[3] = {0, 0, 0}, half = 0.0, max_abs = 0.0;
    if (n) {
        lo[0] = hi[0] = x[0]; lo[1] = hi[1] = y[0]; lo[2] = hi[2] = z[0];
        for (int64_t i = 1; i < n; ++i) {
            if (x[i] < lo[0]) lo[0] = x[i]; if (x[i] > hi[0]) hi[0] = x[i];
            if (y[i] < lo[1]) lo[1] = y[i]; if (y[i] > hi[1]) hi[1] = y[i];
            if (z[i] < lo[2]) lo[2] = z[i]; if (z[i] > hi[2]) hi[2] = z[i];
        }
        double ext = 0.0;
        for (int a = 0; a < 3; ++a) {
            ctr[a] = 0.5 * (lo[a] + hi[a]);
            double e = hi[a] - lo[a];
            if (a == 0 || e > ext) ext = e;
            double m1 = fabs(lo[a]), m2 = fabs(hi[a]);
            if (m1 > max_abs) max_abs = m1;
            if (m2 > max_abs) max_abs = m2;
        }
        half = ext * 0.5;
    }
    t->pad = 8.0 * DBL_EPSILON * (max_abs + half);

    t->cap = 64;
    t->c = malloc(sizeof(double) * 3 * t->cap);
    t->half = malloc(sizeof(double) * t->cap);
    t->child = malloc(sizeof(int64_t) * t->cap);
    t->start = malloc(sizeof(int64_t) * t->cap);
    t->end = malloc(sizeof(int64_t) * t->cap);
    t->perm = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *scratch = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t scap = 1024, sp = 0;
    int64_t *st_node = malloc(sizeof(int64_t) * scap), *st_depth = malloc(sizeof(int64_t) * scap);
    if (!t->c || !t->half || !t->child || !t->start || !t->end || !t->perm || !scratch ||
        !st_node || !st_depth) {
        free(scratch); free(st_node); free(st_depth); otree_free(t); return ST_NOMEM;
    }
    for (int64_t i = 0; i < n; ++i) t->perm[i] = i;
    t->c[0] = ctr[0]; t->c[1] = ctr[1]; t->c[2] = ctr[2];
    t->half[0] = half; t->child[0] = NO_CHILD; t->start[0] = 0; t->end[0] = n;
    t->n_nodes = 1;
    st_node[0] = 0; st_depth[0] = 0; sp = 1;
    int64_t counts[8], offs[9], cursor[8];
    while (sp > 0) {
        --sp;
        int64_t node = st_node[sp], depth = st_depth[sp];
        int64_t s = t->start[node], e = t->end[node];
        if (e - s <= leaf_cap || depth >= max_depth) continue;
        int64_t j0 = t->perm[s];
        int separable = 0;
        for (int64_t q = s + 1; q < e; ++q) {
            int64_t j = t->perm[q];
            if (x[j] != x[j0] || y[j] != y[j0] || z[j] != z[j0]) { separable = 1; break; }
        }
        if (!separable) continue;
        double cx = t->c[3 * node], cy = t->c[3 * node + 1], cz = t->c[3 * node + 2];
        for (int o = 0; o < 8; ++o) counts[o] = 0;
        for (int64_t q = s; q < e; ++q) {
            int64_t j = t->perm[q];
            counts[octant(x[j], y[j], z[j], cx, cy, cz)]++;
        }
        offs[0] = 0;
        for (int o = 0; o < 8; ++o) { offs[o + 1] = offs[o] + counts[o]; cursor[o] = offs[o]; }
        for (int64_t q = s; q < e; ++q) {
            int64_t j = t->perm[q];
            int o = octant(x[j], y[j], z[j], cx, cy, cz);
            scratch[s + cursor[o]] = j;
            cursor[o]++;
        }
        memcpy(t->perm + s, scratch + s, sizeof(int64_t) * (size_t)(e - s));
        if (t->n_nodes + 8 > t->cap && otree_grow(t)) {
            free(scratch); free(st_node); free(st_depth); otree_free(t); return ST_NOMEM;
        }
        int64_t base = t->n_nodes;
        t->child[node] = base;
        double h2 = t->half[node] * 0.5;
        for (int o = 0; o < 8; ++o) {
            int64_t k = base + o;
            t->c[3 * k] = (o & 4) ? cx + h2 : cx - h2;
            t->c[3 * k + 1] = (o & 2) ? cy + h2 : cy - h2;
            t->c[3 * k + 2] = (o & 1) ? cz + h2 : cz - h2;
            t->half[k] = h2;
            t->child[k] = NO_CHILD;
            t->start[k] = s + offs[o];
            t->end[k] = s + offs[o + 1];
        }
        t->n_nodes += 8;
        if (sp + 8 > scap) {
            scap *= 2;
            st_node = realloc(st_node, sizeof(int64_t) * scap);
            st_depth = realloc(st_depth, sizeof(int64_t) * scap);
            if (!st_node || !st_depth) { free(scratch); otree_free(t); return ST_NOMEM; }
        }
        for (int o = 0; o < 8; ++o) {
            int64_t k = base + o;
            if (t->end[k] - t->start[k] > leaf_cap) {
                st_node[sp] = k; st_depth[sp] = depth + 1; ++sp;
            }
        }
    }
    free(scratch); free(st_node); free(st_depth);
    return ST_OK;
}

typedef struct {
    int64_t *idx; double *d2; int64_t cap;
    int64_t *stack; int64_t scap;
} qscratch;

static int qs_init(qscratch *w) {
    w->cap = 8192; w->scap = 4096;
    w->idx = malloc(sizeof(int64_t) * w->cap);
    w->d2 = malloc(sizeof(double) * w->cap);
    w->stack = malloc(sizeof(int64_t) * w->scap);
    return (w->idx && w->d2 && w->stack) ? 0 : -1;
}
static void qs_free(qscratch *w) { free(w->idx); free(w->d2); free(w->stack); }

/* octree.py:179-227; grows its own buffers instead of returning -1/-2 */
static int64_t range_query(const otree *t, qscratch *w, double qx, double qy, double qz,
                           double radius, int64_t exclude) {
    double r2 = radius * radius;
    double rp = radius + t->pad;
    double rp2 = rp * rp;
    int64_t count = 0, sp = 1;
    w->stack[0] = 0;
    const double *x = t->x, *y = t->y, *z = t->z;
    if (t->n == 0) return 0;
    while (sp > 0) {
        int64_t node = w->stack[--sp];
        double h = t->half[node];
        double dx = fabs(qx - t->c[3 * node]) - h; if (dx < 0.0) dx = 0.0;
        double dy = fabs(qy - t->c[3 * node + 1]) - h; if (dy < 0.0) dy = 0.0;
        double dz = fabs(qz - t->c[3 * node + 2]) - h; if (dz < 0.0) dz = 0.0;
        if (dx * dx + dy * dy + dz * dz > rp2) continue;
        int64_t c = t->child[node];
        if (c == NO_CHILD) {
            for (int64_t q = t->start[node]; q < t->end[node]; ++q) {
                int64_t j = t->perm[q];
                if (j == exclude) continue;
                double ddx = x[j] - qx, ddy = y[j] - qy, ddz = z[j] - qz;
                double d2 = ddx * ddx + ddy * ddy + ddz * ddz;
                if (d2 <= r2) {
                    if (count >= w->cap) {
                        w->cap *= 2;
                        w->idx = realloc(w->idx, sizeof(int64_t) * w->cap);
                        w->d2 = realloc(w->d2, sizeof(double) * w->cap);
                        if (!w->idx || !w->d2) return -1;
                    }
                    w->idx[count] = j; w->d2[count] = d2; ++count;
                }
            }
        } else {
            if (sp + 8 > w->scap) {
                w->scap *= 2;
                w->stack = realloc(w->stack, sizeof(int64_t) * w->scap);
                if (!w->stack) return -1;
            }
            for (int o = 0; o < 8; ++o) w->stack[sp++] = c + o;
        }
    }
    return count;
}

/* (d2, index) total order, selection.py:30-32 */
static inline int less_pair(double da, int64_t ia, double db, int64_t ib) {
    return da < db || (da == db && ia < ib);
}
static inline void swap_pair(double *d, int64_t *ix, int64_t a, int64_t b) {
    double td = d[a]; d[a] = d[b]; d[b] = td;
    int64_t ti = ix[a]; ix[a] = ix[b]; ix[b] = ti;
}
static void insertion(double *d, int64_t *ix, int64_t lo, int64_t hi) {
    for (int64_t i = lo + 1; i < hi; ++i) {
        double dv = d[i]; int64_t iv = ix[i]; int64_t j = i - 1;
        while (j >= lo && less_pair(dv, iv, d[j], ix[j])) { d[j + 1] = d[j]; ix[j + 1] = ix[j]; --j; }
        d[j + 1] = dv; ix[j + 1] = iv;
    }
}
static int64_t partition_lomuto(double *d, int64_t *ix, int64_t lo, int64_t hi) {
    int64_t mid = lo + ((hi - lo) >> 1);
    /* median of first/mid/last as pivot, moved to hi-1 */
    int64_t a = lo, b = mid, c = hi - 1;
    if (less_pair(d[b], ix[b], d[a], ix[a])) { int64_t t = a; a = b; b = t; }
    if (less_pair(d[c], ix[c], d[b], ix[b])) { b = c; if (less_pair(d[b], ix[b], d[a], ix[a])) b = a; }
    swap_pair(d, ix, b, hi - 1);
    double pd = d[hi - 1]; int64_t pi = ix[hi - 1];
    int64_t store = lo;
    for (int64_t i = lo; i < hi - 1; ++i)
        if (less_pair(d[i], ix[i], pd, pi)) swap_pair(d, ix, i, store++);
    swap_pair(d, ix, store, hi - 1);
    return store;
}
/* positions [0,k) hold the k smallest under the total order, sorted */
static void select_sorted_prefix(double *d, int64_t *ix, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n, want = k - 1;
    while (hi - lo > 16) {
        int64_t p = partition_lomuto(d, ix, lo, hi);
        if (p == want) break;
        if (want < p) hi = p; else lo = p + 1;
    }
    if (hi - lo <= 16) insertion(d, ix, lo, hi);
    /* sort the prefix; simple iterative quicksort + insertion */
    int64_t st[128][2]; int sp = 0;
    st[sp][0] = 0; st[sp][1] = k; ++sp;
    while (sp > 0) {
        --sp; int64_t l = st[sp][0], h = st[sp][1];
        while (h - l > 16 && sp < 127) {
            int64_t p = partition_lomuto(d, ix, l, h);
            if (p - l < h - p - 1) { st[sp][0] = p + 1; st[sp][1] = h; ++sp; h = p; }
            else { st[sp][0] = l; st[sp][1] = p; ++sp; l = p + 1; }
        }
        insertion(d, ix, l, h);
    }
}

/* kernel.py:30-45 */
static inline double w_lowered(double r, double h) {
    double q = r / h;
    if (q < 1.0) {
        double u = 1.0 - q, u2 = u * u, u4 = u2 * u2;
        return WC6_NORM / (h * h * h) * (u4 * u4 * (1.0 + q * (8.0 + q * (25.0 + 32.0 * q))));
    }
    return 0.0;
}

/* -------------------------------------------------------------------------
 * exported entry points (ctypes; see oracle/__init__.py)
 * ---------------------------------------------------------------------- */

int sph_oracle_perm(int64_t n, const double *x, const double *y, const double *z,
                    int64_t leaf_cap, int64_t *perm_out, int64_t *n_nodes_out) {
    otree t;
    int st = otree_build(&t, n, x, y, z, leaf_cap, 48);
    if (st) return st;
    memcpy(perm_out, t.perm, sizeof(int64_t) * (size_t)n);
    if (n_nodes_out) *n_nodes_out = t.n_nodes;
    otree_free(&t);
    return ST_OK;
}

/* fixed-h neighbour counts: range_query(tree, pos_i, h_i, exclude=i).size */
int sph_oracle_counts(int64_t n, const double *x, const double *y, const double *z,
                      const double *h, int32_t *counts_out, int nthreads) {
    otree t;
    int st = otree_build(&t, n, x, y, z, 8, 48);
    if (st) return st;
    int err = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        qscratch w;
        if (qs_init(&w)) { err = ST_NOMEM; }
        else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 64)
#endif
            for (int64_t i = 0; i < n; ++i) {
                int64_t c = range_query(&t, &w, x[i], y[i], z[i], h[i], i);
                counts_out[i] = (int32_t)c;
            }
        }
        qs_free(&w);
    }
    otree_free(&t);
    (void)nthreads;
    return err;
}

/*
 * The density pass (density.py:286-413) over all particles (targets == NULL)
 * or over a target subset (the sampled-oracle mode of SURVEY 8c(3)): rounds
 * only touch the targets, every target searches the full tree.
 *   h_inout: in = initial smoothing length, out = converged h (targets only)
 *   todo_out[r] = todo size of round r (capacity todo_cap)
 *   info[0] = iterations, info[1] = first degenerate index or -1,
 *   info[2] = still-flagged count on ConvergenceError, info[3] = total
 *   candidates seen (pair tests accepted by the leaf test, all rounds)
 */
/* the todo loop of density.py:286-413 over a built tree (not freed here) */
static int pass_on_tree(otree *tp, int64_t n, const double *x, const double *y, const double *z,
                        const double *mass, double *h_inout, double *rho_out,
                        uint8_t *flags_out, int64_t k, int64_t max_iterations,
                        int nthreads, const int64_t *targets, int64_t n_targets,
                        int64_t *todo_out, int64_t todo_cap, int64_t *info) {
    const double growth = 1.2599210498948732; /* 2.0 ** (1.0 / 3.0), density.py:53 */
    otree t = *tp;
    int64_t nt = targets ? n_targets : n;
    int64_t *todo = malloc(sizeof(int64_t) * (nt ? nt : 1));
    int64_t *next = malloc(sizeof(int64_t) * (nt ? nt : 1));
    if (!todo || !next) { free(todo); free(next); return ST_NOMEM; }
    for (int64_t q = 0; q < nt; ++q) {
        int64_t i = targets ? targets[q] : q;
        todo[q] = i;
        flags_out[i] = 1;
    }
    int64_t ntodo = nt, iteration = 0, cand_total = 0;
    int64_t bad = -1;
    info[0] = 0; info[1] = -1; info[2] = 0; info[3] = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = omp_get_max_threads();
#endif
    while (ntodo > 0) {
        ++iteration;
        if (iteration > max_iterations) {
            info[0] = iteration - 1; info[2] = ntodo; info[3] = cand_total;
            free(todo); free(next);
            return ST_NOT_CONVERGED;
        }
        if (iteration - 1 < todo_cap) todo_out[iteration - 1] = ntodo;
        int err = 0;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads) reduction(+ : cand_total)
#endif
        {
            qscratch w;
            if (qs_init(&w)) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
                err = ST_NOMEM;
            } else {
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 16)
#endif
                for (int64_t q = 0; q < ntodo; ++q) {
                    int64_t i = todo[q];
                    int64_t cnt = range_query(&t, &w, x[i], y[i], z[i], h_inout[i], i);
                    if (cnt < 0) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
                        err = ST_NOMEM;
                        continue;
                    }
                    cand_total += cnt;
                    if (cnt < k) {
                        h_inout[i] = h_inout[i] * growth;
                        flags_out[i] = 1;
                        continue;
                    }
                    select_sorted_prefix(w.d2, w.idx, cnt, k);
                    double hk = sqrt(w.d2[k - 1]);
                    if (hk <= 0.0) {
                        flags_out[i] = 1;
#ifdef _OPENMP
#pragma omp critical(sph_oracle_bad)
#endif
                        { if (bad < 0 || i < bad) bad = i; }
                        continue;
                    }
                    h_inout[i] = hk;
                    flags_out[i] = 0;
                    double rho = mass[i] * w_lowered(0.0, hk);
                    double acc = 0.0;
                    for (int64_t m = 0; m < k; ++m) acc += mass[w.idx[m]] * w_lowered(sqrt(w.d2[m]), hk);
                    rho += acc;
                    rho_out[i] = rho;
                }
            }
            qs_free(&w);
        }
        if (err) { free(todo); free(next); return err; }
        if (bad >= 0) {
            info[0] = iteration; info[1] = bad; info[3] = cand_total;
            free(todo); free(next);
            return ST_DEGENERATE;
        }
        int64_t m = 0;
        for (int64_t q = 0; q < ntodo; ++q) if (flags_out[todo[q]]) next[m++] = todo[q];
        int64_t *tmp = todo; todo = next; next = tmp; ntodo = m;
    }
    info[0] = iteration; info[3] = cand_total;
    free(todo); free(next);
    return ST_OK;
}

int sph_oracle_density_pass(int64_t n, const double *x, const double *y, const double *z,
                            const double *mass, double *h_inout, double *rho_out,
                            uint8_t *flags_out, int64_t k, int64_t max_iterations,
                            int nthreads, const int64_t *targets, int64_t n_targets,
                            int64_t *todo_out, int64_t todo_cap, int64_t *info) {
    if (n <= 0 || k < 1) return ST_INVALID;
    otree t;
    int st = otree_build(&t, n, x, y, z, 8, 48);
    if (st) return st;
    st = pass_on_tree(&t, n, x, y, z, mass, h_inout, rho_out, flags_out, k, max_iterations, nthreads, targets,
                      n_targets, todo_out, todo_cap, info);
    otree_free(&t);
    return st;
}

/* A built tree kept across calls (the CPU baseline times its sampled passes
 * without rebuilding the tree; the positions must outlive the handle). */
void *sph_oracle_tree_new(int64_t n, const double *x, const double *y, const double *z, int *status) {
    otree *t = malloc(sizeof(otree));
    if (!t) { *status = ST_NOMEM; return NULL; }
    *status = n > 0 ? otree_build(t, n, x, y, z, 8, 48) : ST_INVALID;
    if (*status) { free(t); return NULL; }
    return t;
}

void sph_oracle_tree_free(void *h) {
    if (!h) return;
    otree_free((otree *)h);
    free(h);
}

int sph_oracle_density_pass_tree(void *h, const double *mass, double *h_inout, double *rho_out,
                                 uint8_t *flags_out, int64_t k, int64_t max_iterations, int nthreads,
                                 const int64_t *targets, int64_t n_targets, int64_t *todo_out, int64_t todo_cap,
                                 int64_t *info) {
    otree *t = (otree *)h;
    if (!t || k < 1) return ST_INVALID;
    return pass_on_tree(t, t->n, t->x, t->y, t->z, mass, h_inout, rho_out, flags_out, k, max_iterations, nthreads,
                        targets, n_targets, todo_out, todo_cap, info);
}

/* Wendland C6 at separation r for smoothing length h (kernel.py:39-45) */
double sph_oracle_w(double r, double h) { return w_lowered(r, h); }

int sph_oracle_nthreads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

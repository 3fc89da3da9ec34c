/*
 * fmm_oracle.c -- plain, slow, single-threaded fp64 CPU oracle of the 3D Laplace FMM.
 *
 * TEST INFRASTRUCTURE ONLY (see fmm_oracle.h).  Compiled with -O2 -ffp-contract=off so
 * that every floating-point expression is evaluated exactly as written (R7, R8).
 *
 * Rule references (readings listed in DESIGN.md §2):
 *   R1 kernel 1/r, no softening, r^2 == 0 skipped, grad = +grad(phi)   PAPER.md:58 §II-A
 *   R2 root cube, R3 quantisation, R4 63-bit Morton key                 PAPER.md:83 §II-B
 *   R5 stable sort by key (ties by index)                               PAPER.md:92 §II-B
 *   R6 octree: internal iff count > ncrit and level < 21; BFS order
 *   R7 tight boxes, centre, half-diagonal radius                        PAPER.md:94 §II-B
 *   R8 MAC (R_A + R_B) < theta * d, R9 dual tree traversal
 *   R10 canonical lists, R11 coefficient order
 *   R12 P2M, R13 M2M, R14 M2L, R15 L2L, R16 L2P, R17 P2P
 * Nothing here is blocked, fused or reordered beyond what those rules state.
 */
#include "fmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXLEVEL 21

/* ------------------------------------------------------------------ R11 ---- */
/* Multi-indices alpha with |alpha| <= P-1, ordered by degree n, then alpha_x
 * descending, then alpha_y descending. */
typedef struct {
    int P, ncoef;
    int ex[816][3];
    int idx[OFMM_MAXP][OFMM_MAXP][OFMM_MAXP];
} mtab;

static void mtab_init(mtab* t, int P) {
    int k = 0;
    t->P = P;
    for (int n = 0; n < P; ++n)
        for (int a = n; a >= 0; --a)
            for (int b = n - a; b >= 0; --b) {
                int c = n - a - b;
                t->ex[k][0] = a; t->ex[k][1] = b; t->ex[k][2] = c;
                t->idx[a][b][c] = k;
                ++k;
            }
    t->ncoef = k;
}

int ofmm_ncoef(int P) { return P * (P + 1) * (P + 2) / 6; }

void ofmm_multi_index(int P, int idx, int e[3]) {
    mtab t;
    mtab_init(&t, P);
    e[0] = t.ex[idx][0]; e[1] = t.ex[idx][1]; e[2] = t.ex[idx][2];
}

static double factorial(int n) {
    double f = 1.0;
    for (int i = 2; i <= n; ++i) f *= (double)i;
    return f;
}

/* x^e / e! for one axis, by repeated multiplication. */
static double pow_over_fact(double x, int e) {
    double p = 1.0;
    for (int i = 0; i < e; ++i) p *= x;
    return p / factorial(e);
}

/* d^e / e! for a multi-index e. */
static double mono(const double d[3], const int e[3]) {
    return pow_over_fact(d[0], e[0]) * pow_over_fact(d[1], e[1]) * pow_over_fact(d[2], e[2]);
}

/* ------------------------------------------------------------- R2 - R4 ---- */
static void bounds(int64_t n, const double* pos, double lo[3], double hi[3]) {
    for (int d = 0; d < 3; ++d) { lo[d] = pos[d]; hi[d] = pos[d]; }
    for (int64_t i = 1; i < n; ++i)
        for (int d = 0; d < 3; ++d) {
            double x = pos[3 * i + d];
            if (x < lo[d]) lo[d] = x;
            if (x > hi[d]) hi[d] = x;
        }
}

/* R2: c0 = (lo+hi)*0.5, h = 0.5*max_d(hi_d-lo_d) (1 if 0), origin = c0 - h, s = 2^20/h,
 * where lo/hi are the particles' own min/max, or given bounds (the GLOBAL box, so that the
 * local trees of a Morton-range partition are subtrees of one global octree; DESIGN.md §2
 * reading 9). */
static void root_cube_of(const double lo[3], const double hi[3], double o[3], double* scale, double* hout) {
    double c0[3];
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) {
        c0[d] = (lo[d] + hi[d]) * 0.5;
        double e = hi[d] - lo[d];
        if (e > ext) ext = e;
    }
    double h = 0.5 * ext;
    if (h == 0.0) h = 1.0;
    for (int d = 0; d < 3; ++d) o[d] = c0[d] - h;
    *scale = 1048576.0 / h;
    *hout = h;
}

void ofmm_root_cube(int64_t n, const double* pos, double o[3], double* scale, double* hout) {
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    if (n > 0) bounds(n, pos, lo, hi);
    root_cube_of(lo, hi, o, scale, hout);
}

/* R3: i_d = clamp(floor((x_d - o_d) * s), 0, 2^21 - 1). */
static uint32_t quantise(double x, double o, double s) {
    double t = (x - o) * s;
    double f = floor(t);
    if (f < 0.0) return 0u;
    if (f > 2097151.0) return 2097151u;
    return (uint32_t)f;
}

/* R4: digit at level l (1..21) = bit_{21-l}(ix) | bit_{21-l}(iy)<<1 | bit_{21-l}(iz)<<2,
 * key = sum_l digit_l << 3(21-l). */
static uint64_t interleave(uint32_t ix, uint32_t iy, uint32_t iz) {
    uint64_t key = 0;
    for (int l = 1; l <= MAXLEVEL; ++l) {
        int b = MAXLEVEL - l;
        uint64_t digit = (uint64_t)((ix >> b) & 1u) | ((uint64_t)((iy >> b) & 1u) << 1) |
                         ((uint64_t)((iz >> b) & 1u) << 2);
        key |= digit << (3 * (MAXLEVEL - l));
    }
    return key;
}

/* keys under the root cube of `root` (lo xyz, hi xyz) or, when NULL, of the particles' own bounds */
static void keys_in(int64_t n, const double* pos, const double* root, uint64_t* keys) {
    double o[3], s, h;
    if (root) root_cube_of(root, root + 3, o, &s, &h);
    else ofmm_root_cube(n, pos, o, &s, &h);
    for (int64_t i = 0; i < n; ++i)
        keys[i] = interleave(quantise(pos[3 * i], o[0], s), quantise(pos[3 * i + 1], o[1], s),
                             quantise(pos[3 * i + 2], o[2], s));
}

void ofmm_keys(int64_t n, const double* pos, uint64_t* keys) { keys_in(n, pos, NULL, keys); }

/* -------------------------------------------------------------- R12-R17 ---- */
/* R12: M_beta(C) += sum_j q_j (x_j - c)^beta / beta! */
static void p2m_t(const mtab* t, int64_t n, const double* pos, const double* q, const double c[3], double* M) {
    for (int64_t j = 0; j < n; ++j) {
        double d[3] = {pos[3 * j] - c[0], pos[3 * j + 1] - c[1], pos[3 * j + 2] - c[2]};
        for (int b = 0; b < t->ncoef; ++b) M[b] += q[j] * mono(d, t->ex[b]);
    }
}

/* R13: M_alpha(par) += sum_{beta <= alpha} M_beta(ch) s^(alpha-beta)/(alpha-beta)!,  s = c_ch - c_par */
static void m2m_t(const mtab* t, const double* Mc, const double s[3], double* Mp) {
    for (int a = 0; a < t->ncoef; ++a) {
        const int* ea = t->ex[a];
        for (int b = 0; b < t->ncoef; ++b) {
            const int* eb = t->ex[b];
            if (eb[0] > ea[0] || eb[1] > ea[1] || eb[2] > ea[2]) continue;
            int e[3] = {ea[0] - eb[0], ea[1] - eb[1], ea[2] - eb[2]};
            Mp[a] += Mc[b] * mono(s, e);
        }
    }
}

/* R14: Taylor table t_k of 1/|d - y| at y = 0:  t_0 = 1/|d|,
 *   n |d|^2 t_k = (2n-1) sum_i d_i t_{k-e_i} - (n-1) sum_i t_{k-2e_i}   (negative indices omitted),
 * and D^gamma G(d) = (-1)^|gamma| gamma! t_gamma(d). */
static void deriv_t(const mtab* t, const double d[3], double* D) {
    double tk[816];
    double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    tk[0] = 1.0 / sqrt(r2);
    for (int k = 1; k < t->ncoef; ++k) {
        const int* e = t->ex[k];
        int n = e[0] + e[1] + e[2];
        double s1 = 0.0, s2 = 0.0;
        for (int i = 0; i < 3; ++i) {
            if (e[i] >= 1) {
                int m[3] = {e[0], e[1], e[2]};
                m[i] -= 1;
                s1 += d[i] * tk[t->idx[m[0]][m[1]][m[2]]];
            }
            if (e[i] >= 2) {
                int m[3] = {e[0], e[1], e[2]};
                m[i] -= 2;
                s2 += tk[t->idx[m[0]][m[1]][m[2]]];
            }
        }
        tk[k] = ((2.0 * n - 1.0) * s1 - (n - 1.0) * s2) / (n * r2);
    }
    for (int k = 0; k < t->ncoef; ++k) {
        const int* e = t->ex[k];
        int n = e[0] + e[1] + e[2];
        double sign = (n % 2) ? -1.0 : 1.0;
        D[k] = sign * factorial(e[0]) * factorial(e[1]) * factorial(e[2]) * tk[k];
    }
}

/* R14: L_alpha(A) += sum_{|beta| <= P-1-|alpha|} (-1)^|beta| M_beta(B) D^{alpha+beta}G(c_A - c_B) */
static void m2l_t(const mtab* t, const double* M, const double d[3], double* L) {
    double D[816];
    deriv_t(t, d, D);
    for (int a = 0; a < t->ncoef; ++a) {
        const int* ea = t->ex[a];
        int na = ea[0] + ea[1] + ea[2];
        /* beta with |beta| <= P-1-|alpha| are exactly the first ncoef(P-|alpha|) entries (R11) */
        int nbeta = ofmm_ncoef(t->P - na);
        for (int b = 0; b < nbeta; ++b) {
            const int* eb = t->ex[b];
            int nb = eb[0] + eb[1] + eb[2];
            double sign = (nb % 2) ? -1.0 : 1.0;
            L[a] += sign * M[b] * D[t->idx[ea[0] + eb[0]][ea[1] + eb[1]][ea[2] + eb[2]]];
        }
    }
}

/* R15: L_alpha(ch) += sum_{beta >= alpha} L_beta(par) s^(beta-alpha)/(beta-alpha)!,  s = c_ch - c_par */
static void l2l_t(const mtab* t, const double* Lp, const double s[3], double* Lc) {
    for (int a = 0; a < t->ncoef; ++a) {
        const int* ea = t->ex[a];
        for (int b = 0; b < t->ncoef; ++b) {
            const int* eb = t->ex[b];
            if (eb[0] < ea[0] || eb[1] < ea[1] || eb[2] < ea[2]) continue;
            int e[3] = {eb[0] - ea[0], eb[1] - ea[1], eb[2] - ea[2]};
            Lc[a] += Lp[b] * mono(s, e);
        }
    }
}

/* R16: phi_i += sum_alpha L_alpha z^alpha/alpha!;  (grad phi_i)_d += sum_{|g|<=P-2} L_{g+e_d} z^g/g!,
 * z = x_i - c_leaf. */
static void l2p_one(const mtab* t, const double* L, const double c[3], const double* x, double* phi, double* g) {
    double z[3] = {x[0] - c[0], x[1] - c[1], x[2] - c[2]};
    for (int a = 0; a < t->ncoef; ++a) {
        const int* e = t->ex[a];
        double m = mono(z, e);
        *phi += L[a] * m;
        if (e[0] + e[1] + e[2] <= t->P - 2)
            for (int d = 0; d < 3; ++d) {
                int f[3] = {e[0], e[1], e[2]};
                f[d] += 1;
                g[d] += L[t->idx[f[0]][f[1]][f[2]]] * m;
            }
    }
}

/* R17 / R1: phi_i += q_j / r, grad_i += q_j (x_j - x_i) / r^3, skipping r^2 == 0. */
static void p2p_one(const double* xi, int64_t ns, const double* spos, const double* sq, double* phi, double* g) {
    for (int64_t j = 0; j < ns; ++j) {
        double dx = spos[3 * j] - xi[0], dy = spos[3 * j + 1] - xi[1], dz = spos[3 * j + 2] - xi[2];
        double r2 = dx * dx + dy * dy + dz * dz;
        if (r2 == 0.0) continue;
        double r = sqrt(r2);
        double inv = 1.0 / r;
        double inv3 = inv / r2;
        *phi += sq[j] * inv;
        g[0] += sq[j] * dx * inv3;
        g[1] += sq[j] * dy * inv3;
        g[2] += sq[j] * dz * inv3;
    }
}

/* Public single-operator entry points (used by the pins in tests/). */
void ofmm_p2m(int P, int64_t n, const double* pos, const double* q, const double c[3], double* M) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P); p2m_t(t, n, pos, q, c, M); free(t);
}
void ofmm_m2m(int P, const double* Mc, const double s[3], double* Mp) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P); m2m_t(t, Mc, s, Mp); free(t);
}
void ofmm_deriv(int P, const double d[3], double* D) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P); deriv_t(t, d, D); free(t);
}
void ofmm_m2l(int P, const double* M, const double d[3], double* L) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P); m2l_t(t, M, d, L); free(t);
}
void ofmm_l2l(int P, const double* Lp, const double s[3], double* Lc) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P); l2l_t(t, Lp, s, Lc); free(t);
}
void ofmm_l2p(int P, const double* L, const double c[3], int64_t n, const double* pos, double* phi, double* grad) {
    mtab* t = malloc(sizeof(mtab)); mtab_init(t, P);
    for (int64_t i = 0; i < n; ++i) l2p_one(t, L, c, pos + 3 * i, phi + i, grad + 3 * i);
    free(t);
}
void ofmm_p2p(int64_t nt, const double* tpos, int64_t ns, const double* spos, const double* sq,
              double* phi, double* grad) {
    for (int64_t i = 0; i < nt; ++i) p2p_one(tpos + 3 * i, ns, spos, sq, phi + i, grad + 3 * i);
}
void ofmm_direct(int64_t n, const double* pos, const double* q, const int64_t* targets, int64_t nt,
                 double* phi, double* grad) {
    if (!targets) nt = n;
    for (int64_t k = 0; k < nt; ++k) {
        int64_t i = targets ? targets[k] : k;
        phi[k] = 0.0; grad[3 * k] = grad[3 * k + 1] = grad[3 * k + 2] = 0.0;
        p2p_one(pos + 3 * i, n, pos, q, phi + k, grad + 3 * k);
    }
}

/* ------------------------------------------------------------ the method --- */
typedef struct {
    int32_t level;
    uint64_t key;          /* level-l prefix of the particle keys: key >> 3(21-l) */
    uint32_t body_begin, body_count;
    uint32_t child_begin, child_count;
    int32_t parent;
    double bmin[3], bmax[3], c[3], R;
} cell_t;

typedef struct { uint32_t* v; int64_t n, cap; } pairvec;

struct ofmm {
    int64_t n;
    int P, ncrit;
    double theta;
    mtab* t;
    double* pos;   /* sorted positions [n][3] */
    double* q;     /* sorted charges */
    uint64_t* key; /* sorted keys */
    uint32_t* perm;
    cell_t* cells;
    int64_t ncell;
    pairvec m2l, p2p;
    int traversed;
    double *M, *L;
};

typedef struct { uint64_t key; uint32_t idx; } keyidx;

static int cmp_keyidx(const void* a, const void* b) {
    const keyidx* x = a; const keyidx* y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* R6 recursive top-down build into a temporary DFS array. */
typedef struct { cell_t* v; int64_t n, cap; } cellvec;

static int64_t build_rec(ofmm* o, cellvec* cv, int64_t** kids, int32_t level,
                         uint64_t prefix, uint32_t begin, uint32_t count, int32_t parent_dfs) {
    if (cv->n == cv->cap) {
        cv->cap = cv->cap ? 2 * cv->cap : 1024;
        cv->v = realloc(cv->v, cv->cap * sizeof(cell_t));
        *kids = realloc(*kids, cv->cap * 8 * sizeof(int64_t));
    }
    int64_t me = cv->n++;
    cell_t* c = &cv->v[me];
    memset(c, 0, sizeof(*c));
    c->level = level; c->key = prefix; c->body_begin = begin; c->body_count = count;
    c->parent = parent_dfs;
    for (int k = 0; k < 8; ++k) (*kids)[me * 8 + k] = -1;
    if (count > (uint32_t)o->ncrit && level < MAXLEVEL) {
        int shift = 3 * (MAXLEVEL - level - 1);
        uint32_t i = begin, end = begin + count;
        int nc = 0;
        for (int digit = 0; digit < 8; ++digit) {
            uint32_t j = i;
            while (j < end && (int)((o->key[j] >> shift) & 7u) == digit) ++j;
            if (j > i) {
                int64_t child = build_rec(o, cv, kids, level + 1, (prefix << 3) | (uint64_t)digit, i, j - i,
                                          (int32_t)me);
                (*kids)[me * 8 + nc++] = child;
            }
            i = j;
        }
        cv->v[me].child_count = (uint32_t)nc;
    }
    return me;
}

typedef struct { int32_t level; uint64_t key; int64_t dfs; } lvlkey;
static int cmp_lvlkey(const void* a, const void* b) {
    const lvlkey* x = a; const lvlkey* y = b;
    if (x->level != y->level) return x->level < y->level ? -1 : 1;
    return x->key < y->key ? -1 : (x->key > y->key);
}

ofmm* ofmm_create(int64_t n, const double* pos, const double* q, int P, double theta, int ncrit) {
    return ofmm_create_in(n, pos, q, P, theta, ncrit, NULL);
}

ofmm* ofmm_create_in(int64_t n, const double* pos, const double* q, int P, double theta, int ncrit,
                     const double* root) {
    if (n < 0 || P < 1 || P > OFMM_MAXP || !(theta > 0.0 && theta < 1.0) || ncrit < 1) return NULL;
    if (root)
        for (int64_t i = 0; i < n; ++i)
            for (int d = 0; d < 3; ++d)
                if (pos[3 * i + d] < root[d] || pos[3 * i + d] > root[3 + d]) return NULL;   /* outside */
    ofmm* o = calloc(1, sizeof(ofmm));
    o->n = n; o->P = P; o->theta = theta; o->ncrit = ncrit;
    o->t = malloc(sizeof(mtab));
    mtab_init(o->t, P);
    o->pos = malloc((size_t)(3 * n + 1) * sizeof(double));
    o->q = malloc((size_t)(n + 1) * sizeof(double));
    o->key = malloc((size_t)(n + 1) * sizeof(uint64_t));
    o->perm = malloc((size_t)(n + 1) * sizeof(uint32_t));
    if (n == 0) return o; /* R20: no cells */

    /* R2-R4 keys, R5 stable sort (ties by original index) */
    uint64_t* k0 = malloc((size_t)n * sizeof(uint64_t));
    keys_in(n, pos, root, k0);
    keyidx* ki = malloc((size_t)n * sizeof(keyidx));
    for (int64_t i = 0; i < n; ++i) { ki[i].key = k0[i]; ki[i].idx = (uint32_t)i; }
    qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
    for (int64_t i = 0; i < n; ++i) {
        uint32_t j = ki[i].idx;
        o->key[i] = ki[i].key; o->perm[i] = j;
        o->pos[3 * i] = pos[3 * j]; o->pos[3 * i + 1] = pos[3 * j + 1]; o->pos[3 * i + 2] = pos[3 * j + 2];
        o->q[i] = q[j];
    }
    free(ki); free(k0);

    /* R6 recursive build, then canonical (level, key) order */
    cellvec cv = {0};
    int64_t* kids = NULL;
    build_rec(o, &cv, &kids, 0, 0, 0, (uint32_t)n, -1);
    lvlkey* lk = malloc((size_t)cv.n * sizeof(lvlkey));
    for (int64_t i = 0; i < cv.n; ++i) { lk[i].level = cv.v[i].level; lk[i].key = cv.v[i].key; lk[i].dfs = i; }
    qsort(lk, (size_t)cv.n, sizeof(lvlkey), cmp_lvlkey);
    int64_t* bfs_of = malloc((size_t)cv.n * sizeof(int64_t));
    for (int64_t i = 0; i < cv.n; ++i) bfs_of[lk[i].dfs] = i;
    o->ncell = cv.n;
    o->cells = malloc((size_t)cv.n * sizeof(cell_t));
    for (int64_t i = 0; i < cv.n; ++i) {
        int64_t d = lk[i].dfs;
        cell_t c = cv.v[d];
        c.parent = c.parent < 0 ? -1 : (int32_t)bfs_of[c.parent];
        if (c.child_count > 0) {
            c.child_begin = (uint32_t)bfs_of[kids[d * 8]];
            for (uint32_t k = 1; k < c.child_count; ++k) /* children must be contiguous (R6) */
                if (bfs_of[kids[d * 8 + k]] != (int64_t)c.child_begin + k) abort();
        } else {
            c.child_begin = 0;
        }
        o->cells[i] = c;
    }
    free(lk); free(bfs_of); free(kids); free(cv.v);

    /* R7 tight geometry from member particles */
    for (int64_t i = 0; i < o->ncell; ++i) {
        cell_t* c = &o->cells[i];
        const double* p = o->pos + 3 * (size_t)c->body_begin;
        for (int d = 0; d < 3; ++d) { c->bmin[d] = p[d]; c->bmax[d] = p[d]; }
        for (uint32_t j = 1; j < c->body_count; ++j)
            for (int d = 0; d < 3; ++d) {
                double x = p[3 * j + d];
                if (x < c->bmin[d]) c->bmin[d] = x;
                if (x > c->bmax[d]) c->bmax[d] = x;
            }
        double dd[3];
        for (int d = 0; d < 3; ++d) {
            c->c[d] = (c->bmin[d] + c->bmax[d]) * 0.5;
            dd[d] = c->bmax[d] - c->bmin[d];
        }
        c->R = 0.5 * sqrt((dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2]);
    }
    return o;
}

void ofmm_destroy(ofmm* o) {
    if (!o) return;
    free(o->t); free(o->pos); free(o->q); free(o->key); free(o->perm); free(o->cells);
    free(o->m2l.v); free(o->p2p.v); free(o->M); free(o->L);
    free(o);
}

/* ------------------------------------------------------------ R8 - R10 ---- */
static void push_pair(pairvec* v, uint32_t a, uint32_t b) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 4096;
        v->v = realloc(v->v, (size_t)v->cap * 2 * sizeof(uint32_t));
    }
    v->v[2 * v->n] = a; v->v[2 * v->n + 1] = b;
    v->n++;
}

/* R8: accept iff (R_A + R_B) < theta * sqrt((dx*dx + dy*dy) + dz*dz), centre differences. */
static int mac(const ofmm* o, const cell_t* A, const cell_t* B) {
    double dx = A->c[0] - B->c[0], dy = A->c[1] - B->c[1], dz = A->c[2] - B->c[2];
    double d2 = (dx * dx + dy * dy) + dz * dz;
    return (A->R + B->R) < o->theta * sqrt(d2);
}

/* R9 */
static void dtt(ofmm* o, uint32_t a, uint32_t b) {
    const cell_t* A = &o->cells[a];
    const cell_t* B = &o->cells[b];
    int leafA = A->child_count == 0, leafB = B->child_count == 0;
    if (mac(o, A, B)) {
        push_pair(&o->m2l, a, b);
    } else if (leafA && leafB) {
        push_pair(&o->p2p, a, b);
    } else if (leafB || (!leafA && A->R >= B->R)) {
        for (uint32_t k = 0; k < A->child_count; ++k) dtt(o, A->child_begin + k, b);
    } else {
        for (uint32_t k = 0; k < B->child_count; ++k) dtt(o, a, B->child_begin + k);
    }
}

static int cmp_pair(const void* x, const void* y) {
    const uint32_t* a = x; const uint32_t* b = y;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    return a[1] < b[1] ? -1 : (a[1] > b[1]);
}

int ofmm_traverse(ofmm* o) {
    o->m2l.n = 0; o->p2p.n = 0;
    if (o->ncell > 0) dtt(o, 0, 0);
    /* R10: canonical order ascending (target, source); duplicates are impossible */
    if (o->m2l.n) qsort(o->m2l.v, (size_t)o->m2l.n, 2 * sizeof(uint32_t), cmp_pair);
    if (o->p2p.n) qsort(o->p2p.v, (size_t)o->p2p.n, 2 * sizeof(uint32_t), cmp_pair);
    for (int64_t i = 1; i < o->m2l.n; ++i)
        if (cmp_pair(o->m2l.v + 2 * (i - 1), o->m2l.v + 2 * i) >= 0) return -1;
    for (int64_t i = 1; i < o->p2p.n; ++i)
        if (cmp_pair(o->p2p.v + 2 * (i - 1), o->p2p.v + 2 * i) >= 0) return -1;
    o->traversed = 1;
    return 0;
}

/* ------------------------------------------------------------ R12 - R18 --- */
/* post-order upward pass: P2M at leaves, M2M at internal cells */
static void upward(ofmm* o, uint32_t ci) {
    cell_t* c = &o->cells[ci];
    double* M = o->M + (size_t)ci * o->t->ncoef;
    if (c->child_count == 0) {
        p2m_t(o->t, c->body_count, o->pos + 3 * (size_t)c->body_begin, o->q + c->body_begin, c->c, M);
        return;
    }
    for (uint32_t k = 0; k < c->child_count; ++k) {
        uint32_t ch = c->child_begin + k;
        upward(o, ch);
        const cell_t* C = &o->cells[ch];
        double s[3] = {C->c[0] - c->c[0], C->c[1] - c->c[1], C->c[2] - c->c[2]};
        m2m_t(o->t, o->M + (size_t)ch * o->t->ncoef, s, M);
    }
}

/* pre-order downward pass: L2L into children, L2P at leaves */
static void downward(ofmm* o, uint32_t ci, const unsigned char* need, const unsigned char* want_body,
                     double* phi_s, double* grad_s) {
    cell_t* c = &o->cells[ci];
    int nc = o->t->ncoef;
    const double* L = o->L + (size_t)ci * nc;
    if (c->child_count == 0) {
        for (uint32_t j = c->body_begin; j < c->body_begin + c->body_count; ++j)
            if (!want_body || want_body[j]) l2p_one(o->t, L, c->c, o->pos + 3 * (size_t)j, phi_s + j, grad_s + 3 * (size_t)j);
        return;
    }
    for (uint32_t k = 0; k < c->child_count; ++k) {
        uint32_t ch = c->child_begin + k;
        if (need && !need[ch]) continue;
        const cell_t* C = &o->cells[ch];
        double s[3] = {C->c[0] - c->c[0], C->c[1] - c->c[1], C->c[2] - c->c[2]};
        l2l_t(o->t, L, s, o->L + (size_t)ch * nc);
        downward(o, ch, need, want_body, phi_s, grad_s);
    }
}

int ofmm_evaluate(ofmm* o, const int64_t* targets, int64_t nt, double* phi, double* grad) {
    int64_t n = o->n;
    if (!targets) nt = n;
    for (int64_t k = 0; k < nt; ++k) { phi[k] = 0.0; grad[3 * k] = grad[3 * k + 1] = grad[3 * k + 2] = 0.0; }
    if (n == 0) return 0;
    if (!o->traversed && ofmm_traverse(o) != 0) return -1;
    int nc = o->t->ncoef;
    free(o->M); free(o->L);
    o->M = calloc((size_t)o->ncell * nc, sizeof(double));
    o->L = calloc((size_t)o->ncell * nc, sizeof(double));

    /* sampled-target mode: which sorted bodies, which cells (root-to-leaf paths) */
    unsigned char* want_body = NULL;
    unsigned char* need = NULL;
    uint32_t* leaf_of = NULL;
    if (targets) {
        uint32_t* inv = malloc((size_t)n * sizeof(uint32_t));
        for (int64_t i = 0; i < n; ++i) inv[o->perm[i]] = (uint32_t)i;
        want_body = calloc((size_t)n, 1);
        for (int64_t k = 0; k < nt; ++k) {
            if (targets[k] < 0 || targets[k] >= n) { free(inv); free(want_body); return -2; }
            want_body[inv[targets[k]]] = 1;
        }
        free(inv);
        leaf_of = malloc((size_t)n * sizeof(uint32_t));
        need = calloc((size_t)o->ncell, 1);
        for (int64_t ci = 0; ci < o->ncell; ++ci) {
            const cell_t* c = &o->cells[ci];
            if (c->child_count) continue;
            for (uint32_t j = c->body_begin; j < c->body_begin + c->body_count; ++j) leaf_of[j] = (uint32_t)ci;
        }
        for (int64_t j = 0; j < n; ++j)
            if (want_body[j]) {
                int32_t ci = (int32_t)leaf_of[j];
                while (ci >= 0 && !need[ci]) { need[ci] = 1; ci = o->cells[ci].parent; }
            }
    }

    /* 1. upward pass (full: every source multipole is needed) */
    upward(o, 0);
    /* 2. M2L over the list */
    for (int64_t k = 0; k < o->m2l.n; ++k) {
        uint32_t a = o->m2l.v[2 * k], b = o->m2l.v[2 * k + 1];
        if (need && !need[a]) continue;
        const cell_t* A = &o->cells[a];
        const cell_t* B = &o->cells[b];
        double d[3] = {A->c[0] - B->c[0], A->c[1] - B->c[1], A->c[2] - B->c[2]};
        m2l_t(o->t, o->M + (size_t)b * nc, d, o->L + (size_t)a * nc);
    }
    /* 3. P2P over the list, into sorted-order accumulators */
    double* phi_s = calloc((size_t)n, sizeof(double));
    double* grad_s = calloc((size_t)3 * n, sizeof(double));
    for (int64_t k = 0; k < o->p2p.n; ++k) {
        const cell_t* A = &o->cells[o->p2p.v[2 * k]];
        const cell_t* B = &o->cells[o->p2p.v[2 * k + 1]];
        for (uint32_t i = A->body_begin; i < A->body_begin + A->body_count; ++i) {
            if (want_body && !want_body[i]) continue;
            p2p_one(o->pos + 3 * (size_t)i, B->body_count, o->pos + 3 * (size_t)B->body_begin, o->q + B->body_begin,
                    phi_s + i, grad_s + 3 * (size_t)i);
        }
    }
    /* 4. downward pass: L2L, L2P */
    downward(o, 0, need, want_body, phi_s, grad_s);
    /* 5. R18 scatter to caller order */
    if (!targets) {
        for (int64_t i = 0; i < n; ++i) {
            uint32_t j = o->perm[i];
            phi[j] = phi_s[i];
            for (int d = 0; d < 3; ++d) grad[3 * (size_t)j + d] = grad_s[3 * (size_t)i + d];
        }
    } else {
        uint32_t* inv = malloc((size_t)n * sizeof(uint32_t));
        for (int64_t i = 0; i < n; ++i) inv[o->perm[i]] = (uint32_t)i;
        for (int64_t k = 0; k < nt; ++k) {
            uint32_t i = inv[targets[k]];
            phi[k] = phi_s[i];
            for (int d = 0; d < 3; ++d) grad[3 * k + d] = grad_s[3 * (size_t)i + d];
        }
        free(inv);
    }
    free(phi_s); free(grad_s); free(want_body); free(need); free(leaf_of);
    return 0;
}


/* ------------------------------------------------- per-partition mode (§8e) --- */
/* The targets of tree T traversed against the FULL local tree S of another partition, from
 * (root_T, root_S), by the same R8/R9 rules (A from T, B from S).  This is what every rank's
 * remote traversal must reproduce when the LET is sufficient. */
struct ofmm_pairlists { pairvec m2l, p2p; };

static void dtt2(const ofmm* T, const ofmm* S, ofmm_pairlists* out, uint32_t a, uint32_t b) {
    const cell_t* A = &T->cells[a];
    const cell_t* B = &S->cells[b];
    int leafA = A->child_count == 0, leafB = B->child_count == 0;
    if (mac(T, A, B)) {
        push_pair(&out->m2l, a, b);
    } else if (leafA && leafB) {
        push_pair(&out->p2p, a, b);
    } else if (leafB || (!leafA && A->R >= B->R)) {
        for (uint32_t k = 0; k < A->child_count; ++k) dtt2(T, S, out, A->child_begin + k, b);
    } else {
        for (uint32_t k = 0; k < B->child_count; ++k) dtt2(T, S, out, a, B->child_begin + k);
    }
}

ofmm_pairlists* ofmm_traverse_pair(const ofmm* T, const ofmm* S) {
    ofmm_pairlists* pl = calloc(1, sizeof(ofmm_pairlists));
    if (T->ncell > 0 && S->ncell > 0) dtt2(T, S, pl, 0, 0);
    if (pl->m2l.n) qsort(pl->m2l.v, (size_t)pl->m2l.n, 2 * sizeof(uint32_t), cmp_pair);
    if (pl->p2p.n) qsort(pl->p2p.v, (size_t)pl->p2p.n, 2 * sizeof(uint32_t), cmp_pair);
    return pl;
}

void ofmm_pairlists_get(const ofmm_pairlists* pl, int64_t counts[2], uint32_t* m2l, uint32_t* p2p) {
    counts[0] = pl->m2l.n; counts[1] = pl->p2p.n;
    if (m2l && pl->m2l.n) memcpy(m2l, pl->m2l.v, (size_t)pl->m2l.n * 2 * sizeof(uint32_t));
    if (p2p && pl->p2p.n) memcpy(p2p, pl->p2p.v, (size_t)pl->p2p.n * 2 * sizeof(uint32_t));
}

void ofmm_pairlists_free(ofmm_pairlists* pl) {
    if (!pl) return;
    free(pl->m2l.v); free(pl->p2p.v); free(pl);
}

/* phi/grad (caller order of T's particles) with sources = T itself and every S[k]: local
 * lists of T, remote lists (T, S[k]); M of each S[k] from its own upward pass; L2L/L2P in T. */
int ofmm_evaluate_multi(ofmm* T, ofmm* const* S, int nsrc, double* phi, double* grad) {
    int64_t n = T->n;
    for (int64_t k = 0; k < n; ++k) { phi[k] = 0.0; grad[3 * k] = grad[3 * k + 1] = grad[3 * k + 2] = 0.0; }
    if (n == 0) return 0;
    if (!T->traversed && ofmm_traverse(T) != 0) return -1;
    int nc = T->t->ncoef;
    free(T->M); free(T->L);
    T->M = calloc((size_t)T->ncell * nc, sizeof(double));
    T->L = calloc((size_t)T->ncell * nc, sizeof(double));
    upward(T, 0);
    for (int k = 0; k < nsrc; ++k)
        if (S[k]->ncell > 0) {
            free(S[k]->M);
            S[k]->M = calloc((size_t)S[k]->ncell * nc, sizeof(double));
            upward(S[k], 0);
        }
    double* phi_s = calloc((size_t)n, sizeof(double));
    double* grad_s = calloc((size_t)3 * n, sizeof(double));
    for (int k = -1; k < nsrc; ++k) {
        const ofmm* src = k < 0 ? T : S[k];
        ofmm_pairlists* pl = NULL;
        const pairvec* m2l = &T->m2l;
        const pairvec* p2p = &T->p2p;
        if (k >= 0) {
            pl = ofmm_traverse_pair(T, src);
            m2l = &pl->m2l; p2p = &pl->p2p;
        }
        for (int64_t i = 0; i < m2l->n; ++i) {
            const cell_t* A = &T->cells[m2l->v[2 * i]];
            const cell_t* B = &src->cells[m2l->v[2 * i + 1]];
            double d[3] = {A->c[0] - B->c[0], A->c[1] - B->c[1], A->c[2] - B->c[2]};
            m2l_t(T->t, src->M + (size_t)m2l->v[2 * i + 1] * nc, d, T->L + (size_t)m2l->v[2 * i] * nc);
        }
        for (int64_t i = 0; i < p2p->n; ++i) {
            const cell_t* A = &T->cells[p2p->v[2 * i]];
            const cell_t* B = &src->cells[p2p->v[2 * i + 1]];
            for (uint32_t j = A->body_begin; j < A->body_begin + A->body_count; ++j)
                p2p_one(T->pos + 3 * (size_t)j, B->body_count, src->pos + 3 * (size_t)B->body_begin,
                        src->q + B->body_begin, phi_s + j, grad_s + 3 * (size_t)j);
        }
        ofmm_pairlists_free(pl);
    }
    downward(T, 0, NULL, NULL, phi_s, grad_s);
    for (int64_t i = 0; i < n; ++i) {
        uint32_t j = T->perm[i];
        phi[j] = phi_s[i];
        for (int d = 0; d < 3; ++d) grad[3 * (size_t)j + d] = grad_s[3 * (size_t)i + d];
    }
    free(phi_s); free(grad_s);
    return 0;
}

/* -------------------------------------------------------- introspection --- */
void ofmm_counts(const ofmm* o, int64_t c[6]) {
    int64_t nleaf = 0, depth = 0, inter = 0;
    for (int64_t i = 0; i < o->ncell; ++i) {
        if (o->cells[i].child_count == 0) ++nleaf;
        if (o->cells[i].level > depth) depth = o->cells[i].level;
    }
    for (int64_t k = 0; k < o->p2p.n; ++k)
        inter += (int64_t)o->cells[o->p2p.v[2 * k]].body_count * o->cells[o->p2p.v[2 * k + 1]].body_count;
    c[0] = o->ncell; c[1] = nleaf; c[2] = depth; c[3] = o->m2l.n; c[4] = o->p2p.n; c[5] = inter;
}

void ofmm_sorted(const ofmm* o, uint64_t* keys, uint32_t* perm) {
    if (keys) memcpy(keys, o->key, (size_t)o->n * sizeof(uint64_t));
    if (perm) memcpy(perm, o->perm, (size_t)o->n * sizeof(uint32_t));
}

void ofmm_cells(const ofmm* o, int32_t* level, uint64_t* key, uint32_t* bb, uint32_t* bc, uint32_t* cb,
                uint32_t* cc, int32_t* parent, double* bmin, double* bmax, double* center, double* radius) {
    for (int64_t i = 0; i < o->ncell; ++i) {
        const cell_t* c = &o->cells[i];
        if (level) level[i] = c->level;
        if (key) key[i] = c->key;
        if (bb) bb[i] = c->body_begin;
        if (bc) bc[i] = c->body_count;
        if (cb) cb[i] = c->child_begin;
        if (cc) cc[i] = c->child_count;
        if (parent) parent[i] = c->parent;
        for (int d = 0; d < 3; ++d) {
            if (bmin) bmin[3 * i + d] = c->bmin[d];
            if (bmax) bmax[3 * i + d] = c->bmax[d];
            if (center) center[3 * i + d] = c->c[d];
        }
        if (radius) radius[i] = c->R;
    }
}

void ofmm_lists(const ofmm* o, uint32_t* m2l, uint32_t* p2p) {
    if (m2l && o->m2l.n) memcpy(m2l, o->m2l.v, (size_t)o->m2l.n * 2 * sizeof(uint32_t));
    if (p2p && o->p2p.n) memcpy(p2p, o->p2p.v, (size_t)o->p2p.n * 2 * sizeof(uint32_t));
}

void ofmm_expansions(const ofmm* o, double* M, double* L) {
    size_t sz = (size_t)o->ncell * o->t->ncoef * sizeof(double);
    if (M && o->M) memcpy(M, o->M, sz);
    if (L && o->L) memcpy(L, o->L, sz);
}

/*
 * fmm_oracle.h -- plain, slow, single-threaded fp64 CPU oracle of the 3D Laplace FMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1405_7487_b200/, include/fmm.h, libfmm.so) never links, imports or calls it,
 * and the two share no code.
 *
 * What it computes (§II-A, the six operators; §II-C,
 * local tree, post-order P2M/M2M, dual tree traversal, pre-order L2L/L2P), written
 * rule by rule from SURVEY.md §8(c) R1-R20 (the readings are listed in DESIGN.md §2).
 * Every function below cites the rule it follows.
 *
 * Conventions: positions are row-major pos[n][3] doubles, charges q[n]; outputs phi[n],
 * grad[n][3] (grad = +grad phi, R1/Q4); expansions are stored [cell][ncoef] in the
 * graded order of R11.  All functions are pure C, no globals, not thread safe per handle.
 */
#ifndef FMM_ORACLE_H
#define FMM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OFMM_MAXP 16

typedef struct ofmm ofmm;

/* ncoef = P(P+1)(P+2)/6 (R11); exps3 receives the multi-index of coefficient `idx`. */
int  ofmm_ncoef(int P);
void ofmm_multi_index(int P, int idx, int exps3[3]);

/* R2-R4: root cube and 63-bit Morton key of each point (global bounds of the n points). */
void ofmm_root_cube(int64_t n, const double* pos, double origin3[3], double* scale, double* h);
void ofmm_keys(int64_t n, const double* pos, uint64_t* keys);

/* Single operators (R12-R17).  Accumulate (+=) into the output arrays. */
void ofmm_p2m(int P, int64_t n, const double* pos, const double* q, const double c3[3], double* M);
void ofmm_m2m(int P, const double* Mchild, const double shift3[3] /* c_child - c_parent */, double* Mparent);
void ofmm_deriv(int P, const double d3[3], double* D /* D^gamma G(d), ncoef */);
void ofmm_m2l(int P, const double* M, const double d3[3] /* c_A - c_B */, double* L);
void ofmm_l2l(int P, const double* Lparent, const double shift3[3] /* c_child - c_parent */, double* Lchild);
void ofmm_l2p(int P, const double* L, const double c3[3], int64_t n, const double* pos, double* phi, double* grad);
void ofmm_p2p(int64_t nt, const double* tpos, int64_t ns, const double* spos, const double* sq,
              double* phi, double* grad);
/* O(N^2) direct sum (the plain definition, R1) on targets[] (NULL -> all, in order). */
void ofmm_direct(int64_t n, const double* pos, const double* q, const int64_t* targets, int64_t nt,
                 double* phi, double* grad);

/* Whole method.  create: keys, stable sort, recursive tree, geometry (R2-R7).
 * Returns NULL on bad arguments (P outside 1..16, theta outside (0,1), ncrit < 1, n < 0). */
ofmm* ofmm_create(int64_t n, const double* pos, const double* q, int P, double theta, int ncrit);
/* the same with the R2 root cube taken from given bounds root[6] = lo xyz, hi xyz (NULL: the
 * particles' own bounds); NULL result if a particle lies outside them */
ofmm* ofmm_create_in(int64_t n, const double* pos, const double* q, int P, double theta, int ncrit,
                     const double* root);
void  ofmm_destroy(ofmm*);
/* R8-R10: recursive dual tree traversal from (root, root); lists in canonical order. */
int   ofmm_traverse(ofmm*);
/* R12-R18: upward pass, M2L/P2P over the lists, downward pass; outputs in caller order.
 * targets == NULL: every particle (phi[n], grad[n][3]).  Otherwise only those original
 * indices (phi[nt], grad[nt][3] in the order of targets[]); M2L/L2L/L2P/P2P are then
 * applied only on the root-to-leaf paths of the target leaves (sampled-target mode). */
int   ofmm_evaluate(ofmm*, const int64_t* targets, int64_t nt, double* phi, double* grad);

/* Introspection, canonical orders (R5, R6, R10).
 * counts: [0]=ncell [1]=nleaf [2]=depth [3]=n_m2l [4]=n_p2p [5]=p2p body-pair interactions */
void ofmm_counts(const ofmm*, int64_t counts[6]);
void ofmm_sorted(const ofmm*, uint64_t* keys, uint32_t* perm);
void ofmm_cells(const ofmm*, int32_t* level, uint64_t* key, uint32_t* body_begin, uint32_t* body_count,
                uint32_t* child_begin, uint32_t* child_count, int32_t* parent,
                double* bmin3, double* bmax3, double* center3, double* radius);
void ofmm_lists(const ofmm*, uint32_t* m2l /* [n_m2l][2] */, uint32_t* p2p /* [n_p2p][2] */);
void ofmm_expansions(const ofmm*, double* M, double* L);   /* [ncell][ncoef] each; NULL to skip */

/* Per-partition mode: the targets of tree T against the full local tree S
 * of another partition, from (root_T, root_S) under R8-R10; and phi/grad of T's particles with
 * sources T and S[0..nsrc).  Each tree is built from its own particles (local root cube,
 * PAPER.md:118 §II-C "completely local construction of the octree using the local bounding box"). */
typedef struct ofmm_pairlists ofmm_pairlists;
ofmm_pairlists* ofmm_traverse_pair(const ofmm* T, const ofmm* S);
void ofmm_pairlists_get(const ofmm_pairlists*, int64_t counts[2], uint32_t* m2l, uint32_t* p2p);
void ofmm_pairlists_free(ofmm_pairlists*);
int  ofmm_evaluate_multi(ofmm* T, ofmm* const* S, int nsrc, double* phi, double* grad);

#ifdef __cplusplus
}
#endif
#endif

/* tpdg oracle: CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the checker the parity tests, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg compare the CUDA path against. It is never linked into,
 * loaded by, or called from the product library (paper_1704_04549_b200/).
 *
 * Every function restates one reference function (cited file:line into
 * /root/reference/proj/include/tpdg/) in plain C with the reference's
 * summation order; built with -ffp-contract=off it reproduces the reference
 * built with its own CMake Release flags bit for bit (pinned against the
 * golden fixtures in tests/golden/, produced by oracle/ref_driver.cpp).
 *
 * Layouts are the reference's:
 *   vectors   [e][c][tensor index, x fastest]                 (ops/state.hpp:12-13)
 *   g, d      mu x q row-major; gw, dw q x mu                   (dg/reference_element.hpp:24-27)
 *   jdet      [e][mu^d]; face_w [e][2d][mu^(d-1)]               (dg/mesh.hpp:87-92)
 *   conn      [e][2d][3] = neighbor, neighbor_face, orientation (dg/mesh.hpp:37-42)
 *   dft       [e][dir][qv][r][c]; dfm, dfp [e][f][qf][r][c]     (ops/linearized.hpp:15-33)
 */
#ifndef TPDG_ORACLE_H
#define TPDG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dim, n_c, q, mu, n_elements;
  const double *g, *d, *gw, *dw, *w;
  const double *jdet, *face_w;
  const int64_t *conn;
  const double *dft, *dfm, *dfp;
} or_sys;

enum { OR_OK = 0, OR_SINGULAR = 1, OR_CONVERGENCE = 2, OR_SHAPE = 3 };

/* libstdc++ <random> restated: mt19937_64 + uniform_real / normal (polar). */
void or_uniform_vector(uint64_t seed, long n, double scale, double *out);
void or_seeded_unit_vector(long n, uint64_t seed, double *out);

/* ops */
void or_elem_diag_apply(const or_sys *s, int e, double a, double b, int small_mode, const double *vin,
                        double *vout);
void or_jv(const or_sys *s, double a, double b, int small_mode, const double *vin, double *vout);
void or_shuffled(const or_sys *s, int e, double a, double b, int small_mode, int comp, int transpose,
                 const double *in, double *out);
void or_assemble_block(const or_sys *s, int e, double a, double b, int small_mode, int comp, double *blk);

/* small dense linear algebra */
int or_lu_factor(int n, const double *a, double *lu, int *perm);
void or_lu_solve(int n, const double *lu, const int *perm, const double *b, double *x);
int or_real_schur(int n, const double *c, double *q, double *t);
int or_sylvester(int n1, int n2, const double *t1, const double *t2, const double *b, double *x);
void or_svd_small(int m, int n, const double *a, double *u, double *sigma, double *v);

/* KSVD preconditioner */
typedef struct or_pc or_pc;
or_pc *or_form_ksvd(const or_sys *s, double a, double b, int small_mode, int terms, const double *start_vec,
                    const double *start_vec2);
void or_pc_free(or_pc *pc);
int or_pc_num_fallbacks(const or_pc *pc);
void or_pc_fallbacks(const or_pc *pc, int64_t *out); /* pairs (element, component) */
int or_pc_has_factors(const or_pc *pc, int blk);
/* 2D: a1 b1 a2 b2 ; 3D: a1 b1 c1 b2 c2 (row-major, concatenated) */
void or_pc_factors(const or_pc *pc, int blk, double *out);
/* formed apply state of one block: LU factors then Schur pairs (Q1 T1 Q2 T2), and the pivots */
int or_pc_record_len(const or_pc *pc);
int or_pc_piv_len(const or_pc *pc);
void or_pc_record(const or_pc *pc, int blk, double *rec, int *piv);
int or_pc_factor_len(const or_pc *pc);
void or_pc_apply(const or_pc *pc, const double *in, double *out);
/* 2D apply of given factors (reference ksvd.hpp:75-129), rhs overwritten */
int or_apply_factors_2d(int n1, int n2, const double *a1, const double *b1, const double *a2, const double *b2,
                        double *x);

/* Restarted right/left-preconditioned GMRES (reference solve/gmres.hpp:52-179). */
int or_gmres(const or_sys *s, double a, double b, int small_mode, const or_pc *pc, const double *rhs, double tol,
             int restart, int max_it, int left, double *x, int *iterations, double *hist, int hist_cap,
             int *converged);

#ifdef __cplusplus
}
#endif
#endif

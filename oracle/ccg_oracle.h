/*
 * ccg_oracle.h -- CPU restatement of the reference cCG solver and of the
 * BASELINE input generators.  TEST INFRASTRUCTURE ONLY (see ccg_oracle.c).
 */
#ifndef COOPCG_ORACLE_H
#define COOPCG_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COOPCG_ORACLE_MAX_P 64

enum { ORC_OK = 0, ORC_E_DIMENSION = 1, ORC_E_SPD_VIOLATION = 2, ORC_E_NUMERICAL_BREAKDOWN = 3 };
enum { ORC_STATUS_CONVERGED = 0, ORC_STATUS_RANK_COLLAPSE = 1, ORC_STATUS_MAX_ITERATIONS = 2 };

typedef struct {
    double tol;
    int max_iters;
    int recompute_residual_every;
    double rank_rel_tol;
} orc_opts;

typedef struct {
    int status;
    int converged_agent;
    int iterations;
    int capacity;                  /* rows the per-iteration arrays hold */
    double* residual_norms;        /* [capacity * p], may be NULL */
    double* minres;                /* [capacity], may be NULL */
    uint64_t* wall_ns;             /* [capacity], may be NULL */
    double* initial_residual_norms;/* [p], may be NULL */
    double initial_minres;
    double* final_x;               /* [n * p] column-major, may be NULL */
    double* final_residual_norms;  /* [p], may be NULL */
    double final_minres;
    uint64_t loop_wall_ns;
    char error_msg[256];
    int* active_agents;            /* [p], may be NULL: surviving agent ids */
    int n_active;
} orc_trace;

double orc_dot(const double* a, const double* b, long n);
void orc_matvec_col(const double* A, int n, const double* d, double* out);
void orc_matvec_block(const double* A, int n, const double* D, int p, double* out);
int orc_lu_factor(double* m, int p, int* perm, double pivot_floor);
void orc_lu_solve_vec(const double* lu, int p, const int* perm, const double* rhs, double* x);
void orc_gram(const double* D, const double* AD, int n, int p, double* raw, double* sym);
int orc_solve_small(const double* M, int p, const double* B, int q, double* X);
int orc_numerical_rank(const double* D, int n, int p, double tol, int* columns);
int orc_ccg_solve(int n, int p, const double* A, const double* b, const double* X0,
                  const orc_opts* opts, orc_trace* tr);
int orc_mccg_solve(int n, int p, const double* A, const double* b, const double* X0,
                   const orc_opts* opts, orc_trace* tr);
int orc_block_solve(int n, int p, const double* A, const double* b, const double* X0,
                    const orc_opts* opts, int allow_restriction, orc_trace* tr);

/* BASELINE generators, restated independently of the product (gen_oracle.c). */
void orc_gen_diagdom(int n, uint64_t seed, double* A);
void orc_gen_householder_factors(int n, int m, double kappa, uint64_t seed, double* V,
                                 double* lambda);
void orc_gen_householder(int n, int m, const double* V, const double* lambda, double* A);
void orc_gen_diagdom_rows(int n, uint64_t seed, int r0, int r1, double* out);
void orc_gen_householder_par(int n, int m, const double* V, const double* lambda, double* A);
void orc_gen_rhs(int n, int kind, uint64_t seed, double* b);
void orc_gen_starts(int n, int p, uint64_t seed, double* X0_colmajor);

#ifdef __cplusplus
}
#endif
#endif

/*
 * ccg_oracle.c -- CPU restatement of the reference cooperative-CG solver.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1204_0069_b200/,
 * include/, the CUDA library) may link or call this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
 * the checker.
 *
 * This is an independent plain-C restatement of the reference's float-mode
 * `ccg_solve` (coopcg/solvers.hpp:329-333), following its operation order
 * exactly so results are bit-identical:
 *   - ascending-index accumulation starting from +0.0, one rounding per
 *     multiply and per add (no FMA: build with -ffp-contract=off, as the
 *     reference does, CMakeLists.txt:25);
 *   - the stage order of drive() (solvers.hpp:259-283).
 * Parity pin: tests/test_oracle.py checks this file bit-for-bit against the
 * reference itself (oracle/_ref, compiled from /root/reference by
 * oracle/build_ref.sh) and against the committed golden fixtures in
 * tests/golden/ that the reference produced.
 *
 * Layouts follow the reference: A n x n row-major (dense.hpp:101-170), blocks
 * n x p column-major (dense.hpp:35-38), p x p grids row-major
 * (block_cg.hpp:45-46).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "ccg_oracle.h"

/* kernels.hpp:20-26 -- acc = +0.0; acc += a[k]*b[k], k ascending. */
double orc_dot(const double* a, const double* b, long n) {
    double acc = 0.0;
    for (long k = 0; k < n; ++k) acc += a[k] * b[k];
    return acc;
}

/* kernels.hpp:28-34 -- out[i] = dot(A.row(i), d). */
void orc_matvec_col(const double* A, int n, const double* d, double* out) {
    for (int i = 0; i < n; ++i) out[i] = orc_dot(A + (size_t)i * n, d, n);
}

/* dense_ops.hpp:16-25 -- A * D column by column (D, out column-major). */
void orc_matvec_block(const double* A, int n, const double* D, int p, double* out) {
    for (int j = 0; j < p; ++j) orc_matvec_col(A, n, D + (size_t)j * n, out + (size_t)j * n);
}

/* kernels.hpp:36-49 -- dest[i] = base[i] + sum_j coeff[j]*B(i,j), j ascending. */
static void combine_columns(double* dest, const double* base, const double* B, int n, int p,
                            const double* coeff) {
    for (int i = 0; i < n; ++i) {
        double acc = base[i];
        for (int j = 0; j < p; ++j) acc += coeff[j] * B[(size_t)j * n + i];
        dest[i] = acc;
    }
}

/* kernels.hpp:61-95 -- LU with partial pivoting, largest |.|, lowest row on
 * ties; fails when the chosen pivot is not above the floor. */
int orc_lu_factor(double* m, int p, int* perm, double pivot_floor) {
    for (int i = 0; i < p; ++i) perm[i] = i;
    for (int k = 0; k < p; ++k) {
        int piv = k;
        double best = fabs(m[(size_t)k * p + k]);
        for (int i = k + 1; i < p; ++i) {
            double cand = fabs(m[(size_t)i * p + k]);
            if (cand > best) {
                best = cand;
                piv = i;
            }
        }
        if (!(best > pivot_floor)) return 0;
        if (piv != k) {
            for (int j = 0; j < p; ++j) {
                double t = m[(size_t)k * p + j];
                m[(size_t)k * p + j] = m[(size_t)piv * p + j];
                m[(size_t)piv * p + j] = t;
            }
            int t = perm[k];
            perm[k] = perm[piv];
            perm[piv] = t;
        }
        for (int i = k + 1; i < p; ++i) {
            const double mult = m[(size_t)i * p + k] / m[(size_t)k * p + k];
            m[(size_t)i * p + k] = mult;
            for (int j = k + 1; j < p; ++j) m[(size_t)i * p + j] -= mult * m[(size_t)k * p + j];
        }
    }
    return 1;
}

/* kernels.hpp:97-115 -- forward then backward substitution. */
void orc_lu_solve_vec(const double* lu, int p, const int* perm, const double* rhs, double* x) {
    double y[COOPCG_ORACLE_MAX_P];
    for (int i = 0; i < p; ++i) {
        double acc = rhs[perm[i]];
        for (int j = 0; j < i; ++j) acc -= lu[(size_t)i * p + j] * y[j];
        y[i] = acc;
    }
    for (int i = p - 1; i >= 0; --i) {
        double acc = y[i];
        for (int j = i + 1; j < p; ++j) acc -= lu[(size_t)i * p + j] * x[j];
        x[i] = acc / lu[(size_t)i * p + i];
    }
}

/* block_cg.hpp:180-190 / dense_ops.hpp:62-72 -- max|M| * 1e-14. */
static double pivot_floor_of(const double* m, int p) {
    double maxabs = 0.0;
    for (int t = 0; t < p * p; ++t) {
        double v = fabs(m[t]);
        maxabs = (maxabs < v) ? v : maxabs; /* std::max(a,b) = (a<b)?b:a */
    }
    return maxabs * 1e-14;
}

/* dense_ops.hpp:30-56 -- raw(i,j)=dot(D_i, AD_j); gram = (raw+raw^T)/2. */
void orc_gram(const double* D, const double* AD, int n, int p, double* raw, double* sym) {
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
            raw[(size_t)i * p + j] = orc_dot(D + (size_t)i * n, AD + (size_t)j * n, n);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
            sym[(size_t)i * p + j] = (raw[(size_t)i * p + j] + raw[(size_t)j * p + i]) / 2.0;
}

/* dense_ops.hpp:62-92 -- solve M X = B (B p x q column-major) by one LU.
 * Returns 0 when a pivot vanished (SingularMatrixError). */
int orc_solve_small(const double* M, int p, const double* B, int q, double* X) {
    double lu[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    int perm[COOPCG_ORACLE_MAX_P];
    memcpy(lu, M, sizeof(double) * (size_t)p * p);
    if (!orc_lu_factor(lu, p, perm, pivot_floor_of(M, p))) return 0;
    for (int j = 0; j < q; ++j) orc_lu_solve_vec(lu, p, perm, B + (size_t)j * p, X + (size_t)j * p);
    return 1;
}

/* dense_ops.hpp:104-157 -- numerical rank by column-pivoted MGS on squared
 * norms; a step is accepted while best_sq > tol^2 * (first pivot sq).
 * `columns` (may be NULL) receives the chosen column indices in order. */
int orc_numerical_rank(const double* D, int n, int p, double tol, int* columns) {
    if (n == 0 || p == 0) return 0;
    double* V = (double*)malloc(sizeof(double) * (size_t)n * p);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(V, D, sizeof(double) * (size_t)n * p);
    int used[COOPCG_ORACLE_MAX_P] = {0};
    int rank = 0;
    double max_pivot_sq = 0.0;
    const double tol_sq = tol * tol;
    for (int step = 0; step < p; ++step) {
        int best = -1;
        double best_sq = 0.0;
        for (int j = 0; j < p; ++j) {
            if (used[j]) continue;
            const double nsq = orc_dot(V + (size_t)j * n, V + (size_t)j * n, n);
            if (best < 0 || nsq > best_sq) {
                best = j;
                best_sq = nsq;
            }
        }
        if (step == 0) max_pivot_sq = best_sq;
        if (!(best_sq > tol_sq * max_pivot_sq)) break;
        used[best] = 1;
        if (columns) columns[rank] = best;
        ++rank;
        memcpy(q, V + (size_t)best * n, sizeof(double) * (size_t)n);
        const double qsq = best_sq;
        for (int j = 0; j < p; ++j) {
            if (used[j]) continue;
            double* c = V + (size_t)j * n;
            const double coef = orc_dot(q, c, n) / qsq;
            for (int i = 0; i < n; ++i) c[i] -= coef * q[i];
        }
    }
    free(V);
    free(q);
    return rank;
}

static uint64_t now_ns(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

/* block_cg.hpp:297-303 -- m = norms[0]; m = std::min(m, v) over all. */
static double min_norm(const double* v, int p) {
    double m = p > 0 ? v[0] : 0.0;
    for (int j = 0; j < p; ++j) m = (v[j] < m) ? v[j] : m;
    return m;
}

/* block_cg.hpp:305-311 -- first slot with ||r_j|| <= tol, else -1. */
static int first_converged(const double* norms, int p, double tol) {
    for (int j = 0; j < p; ++j)
        if (norms[j] <= tol) return j;
    return -1;
}

/* One residual recomputation: r = A x - b (block_cg.hpp:132-138, :236-241). */
static void residual_of(const double* A, const double* b, int n, const double* x, double* r) {
    orc_matvec_col(A, n, x, r);
    for (int i = 0; i < n; ++i) r[i] -= b[i];
}

/* BlockCgWorkspace::restrict_to (block_cg.hpp:84-96): keep the listed slots
 * (ascending) of the n x p column-major blocks. */
static void keep_columns(double* blk, int n, const int* keep, int pk) {
    for (int c = 0; c < pk; ++c)
        if (keep[c] != c) memmove(blk + (size_t)c * n, blk + (size_t)keep[c] * n, sizeof(double) * n);
}

static int cmp_int(const void* a, const void* b) { return *(const int*)a - *(const int*)b; }

/*
 * The serial block driver: run_serial_block (solvers.hpp:308-321) with
 * drive() (solvers.hpp:259-283).  allow_restriction = 0 is ccg_solve
 * (solvers.hpp:329-333), 1 is mccg_solve (solvers.hpp:338-342).  Per-iteration
 * norms are written per ORIGINAL agent id (NaN for agents no longer active);
 * final_x / final_residual_norms likewise (NaN columns for dropped agents).
 */
int orc_block_solve(int n, int p, const double* A, const double* b, const double* X0,
                    const orc_opts* opts, int allow_restriction, orc_trace* tr) {
    tr->status = ORC_STATUS_MAX_ITERATIONS;
    tr->converged_agent = -1;
    tr->iterations = 0;
    tr->loop_wall_ns = 0;
    tr->error_msg[0] = '\0';
    /* solvers.hpp:300-306 */
    if (n <= 0 || p < 1 || p >= n || p > COOPCG_ORACLE_MAX_P) {
        snprintf(tr->error_msg, sizeof tr->error_msg,
                 "solver: need 1 <= p < n starting columns");
        return ORC_E_DIMENSION;
    }
    const size_t np = (size_t)n * p;
    const int max_iters = opts->max_iters >= 0 ? opts->max_iters : 2 * n; /* solvers.hpp:18-23 */
    const int every = opts->recompute_residual_every >= 0 ? opts->recompute_residual_every : 50;
    double* X = (double*)malloc(sizeof(double) * np);
    double* R = (double*)malloc(sizeof(double) * np);
    double* D = (double*)malloc(sizeof(double) * np);
    double* Dn = (double*)malloc(sizeof(double) * np);
    double* AD = (double*)malloc(sizeof(double) * np);
    double gram_raw[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    double gram[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    double rhs[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    double alpha[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    double beta[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    double lu[COOPCG_ORACLE_MAX_P * COOPCG_ORACLE_MAX_P];
    int perm[COOPCG_ORACLE_MAX_P];
    double nsq[COOPCG_ORACLE_MAX_P], norm[COOPCG_ORACLE_MAX_P];
    int rc = ORC_OK;
    int ids[COOPCG_ORACLE_MAX_P];
    const int p0 = p;
    for (int j = 0; j < p; ++j) ids[j] = j;
    memcpy(X, X0, sizeof(double) * np);

    /* stage_setup (block_cg.hpp:132-144): R = A X - b, D = R, norms. */
    for (int i = 0; i < p; ++i) {
        residual_of(A, b, n, X + (size_t)i * n, R + (size_t)i * n);
        memcpy(D + (size_t)i * n, R + (size_t)i * n, sizeof(double) * n);
        nsq[i] = orc_dot(R + (size_t)i * n, R + (size_t)i * n, n);
        norm[i] = sqrt(nsq[i]);
    }
    /* setup_coordinator (solvers.hpp:55-100) */
    int stop = 0;
    if (tr->initial_residual_norms) memcpy(tr->initial_residual_norms, norm, sizeof(double) * p);
    tr->initial_minres = min_norm(norm, p);
    {
        int cols[COOPCG_ORACLE_MAX_P];
        const int rank0 = orc_numerical_rank(D, n, p, opts->rank_rel_tol, cols);
        if (allow_restriction && rank0 > 0 && rank0 < p) {  /* solvers.hpp:67-76 */
            qsort(cols, rank0, sizeof(int), cmp_int);
            keep_columns(X, n, cols, rank0);
            keep_columns(R, n, cols, rank0);
            keep_columns(D, n, cols, rank0);
            int nid[COOPCG_ORACLE_MAX_P];
            for (int c = 0; c < rank0; ++c) nid[c] = ids[cols[c]];
            memcpy(ids, nid, sizeof(int) * rank0);
            p = rank0;
            for (int j = 0; j < p; ++j) {
                nsq[j] = orc_dot(R + (size_t)j * n, R + (size_t)j * n, n);
                norm[j] = sqrt(nsq[j]);
            }
        }
        const int slot = first_converged(norm, p, opts->tol);
        if (slot >= 0) {
            tr->status = ORC_STATUS_CONVERGED;
            tr->converged_agent = ids[slot];
            stop = 1;
        } else if (!allow_restriction && rank0 < p) {
            tr->status = ORC_STATUS_RANK_COLLAPSE;
            stop = 1;
        } else if (allow_restriction && rank0 == 0) {      /* solvers.hpp:86-91 */
            snprintf(tr->error_msg, sizeof tr->error_msg, "every starting direction is numerically zero");
            rc = ORC_E_NUMERICAL_BREAKDOWN;
            stop = 1;
        }
        if (!stop && max_iters == 0) {
            tr->status = ORC_STATUS_MAX_ITERATIONS;
            stop = 1;
        }
    }
    int k = 0;
    uint64_t t_iter = now_ns();
    while (!stop) {
        /* stage_matvec (block_cg.hpp:146-151) */
        orc_matvec_block(A, n, D, p, AD);
        /* stage_gram_row + stage_gram_finalize (block_cg.hpp:153-178) */
        orc_gram(D, AD, n, p, gram_raw, gram);
        /* stage_alpha (block_cg.hpp:193-218): SPD guard, rhs, LU, solve. */
        int spd_failed = 0, rank_failed = 0;
        for (int i = 0; i < p; ++i) {
            const double dm = gram[(size_t)i * p + i];
            if (!(dm > 0.0) && orc_dot(D + (size_t)i * n, D + (size_t)i * n, n) > 0.0) {
                spd_failed = 1;
                continue;
            }
            for (int j = 0; j < p; ++j)
                rhs[(size_t)i * p + j] = -orc_dot(R + (size_t)i * n, D + (size_t)j * n, n);
            memcpy(lu, gram, sizeof(double) * (size_t)p * p);
            if (!orc_lu_factor(lu, p, perm, pivot_floor_of(gram, p))) {
                rank_failed = 1;
                continue;
            }
            orc_lu_solve_vec(lu, p, perm, rhs + (size_t)i * p, alpha + (size_t)i * p);
        }
        if (!spd_failed && !rank_failed) {
            /* stage_update (block_cg.hpp:222-244) */
            const int recompute = every > 0 && (k + 1) % every == 0; /* solvers.hpp:33-35 */
            for (int i = 0; i < p; ++i) {
                double* ri = R + (size_t)i * n;
                double* xi = X + (size_t)i * n;
                const double* ai = alpha + (size_t)i * p;
                if (!recompute) {
                    combine_columns(ri, ri, AD, n, p, ai);
                    combine_columns(xi, xi, D, n, p, ai);
                } else {
                    combine_columns(xi, xi, D, n, p, ai);
                    residual_of(A, b, n, xi, ri);
                }
            }
            /* stage_beta (block_cg.hpp:248-266) */
            for (int i = 0; i < p; ++i) {
                for (int j = 0; j < p; ++j)
                    rhs[(size_t)i * p + j] = -orc_dot(R + (size_t)i * n, AD + (size_t)j * n, n);
                memcpy(lu, gram, sizeof(double) * (size_t)p * p);
                if (!orc_lu_factor(lu, p, perm, pivot_floor_of(gram, p))) {
                    rank_failed = 1;
                    continue;
                }
                orc_lu_solve_vec(lu, p, perm, rhs + (size_t)i * p, beta + (size_t)i * p);
            }
        }
        if (!spd_failed && !rank_failed) {
            /* stage_direction_and_norms (block_cg.hpp:270-277) */
            for (int i = 0; i < p; ++i) {
                combine_columns(Dn + (size_t)i * n, R + (size_t)i * n, D, n, p, beta + (size_t)i * p);
                nsq[i] = orc_dot(R + (size_t)i * n, R + (size_t)i * n, n);
                norm[i] = sqrt(nsq[i]);
            }
        }
        /* end_of_iteration (solvers.hpp:102-185) */
        const uint64_t wall = now_ns() - t_iter;
        if (spd_failed) {
            snprintf(tr->error_msg, sizeof tr->error_msg,
                     "nonpositive direction energy d^T A d at iteration %d", k);
            rc = ORC_E_SPD_VIOLATION;
            break;
        }
        if (rank_failed) {
            tr->status = ORC_STATUS_RANK_COLLAPSE;
            break;
        }
        if (k < tr->capacity) {
            if (tr->residual_norms) {
                for (int j = 0; j < p0; ++j) tr->residual_norms[(size_t)k * p0 + j] = NAN;
                for (int j = 0; j < p; ++j) tr->residual_norms[(size_t)k * p0 + ids[j]] = norm[j];
            }
            if (tr->minres) tr->minres[k] = min_norm(norm, p);
            if (tr->wall_ns) tr->wall_ns[k] = wall;
        }
        tr->iterations = k + 1;
        tr->loop_wall_ns += wall;
        const int slot = first_converged(norm, p, opts->tol);
        if (slot >= 0) {
            tr->status = ORC_STATUS_CONVERGED;
            tr->converged_agent = ids[slot];
            break;
        }
        {
            const int rr = orc_numerical_rank(Dn, n, p, opts->rank_rel_tol, NULL);
            if (rr < p) {                                   /* solvers.hpp:156-175 */
                if (!allow_restriction) {
                    tr->status = ORC_STATUS_RANK_COLLAPSE;
                    break;
                }
                int cols[COOPCG_ORACLE_MAX_P];
                const int nsel = orc_numerical_rank(R, n, p, opts->rank_rel_tol, cols);
                const int pnext = rr < nsel ? rr : nsel;
                if (pnext == 0) {
                    snprintf(tr->error_msg, sizeof tr->error_msg,
                             "all agents degenerate at iteration %d with residual above tolerance", k);
                    rc = ORC_E_NUMERICAL_BREAKDOWN;
                    break;
                }
                qsort(cols, pnext, sizeof(int), cmp_int);
                keep_columns(X, n, cols, pnext);
                keep_columns(R, n, cols, pnext);
                keep_columns(Dn, n, cols, pnext);
                int nid[COOPCG_ORACLE_MAX_P];
                for (int c = 0; c < pnext; ++c) nid[c] = ids[cols[c]];
                memcpy(ids, nid, sizeof(int) * pnext);
                p = pnext;
            }
        }
        if (k + 1 >= max_iters) {
            tr->status = ORC_STATUS_MAX_ITERATIONS;
            break;
        }
        double* t = D;
        D = Dn;
        Dn = t;
        ++k;
        t_iter = now_ns();
    }
    /* finalize_trace (solvers.hpp:188-210): true residuals of the final X. */
    if (tr->final_x) {
        for (size_t e = 0; e < (size_t)n * p0; ++e) tr->final_x[e] = NAN;
        for (int j = 0; j < p; ++j) memcpy(tr->final_x + (size_t)ids[j] * n, X + (size_t)j * n, sizeof(double) * n);
    }
    if (tr->active_agents) {
        for (int j = 0; j < p; ++j) tr->active_agents[j] = ids[j];
    }
    tr->n_active = p;
    {
        double fr[COOPCG_ORACLE_MAX_P];
        for (int j = 0; j < p; ++j) {
            residual_of(A, b, n, X + (size_t)j * n, AD); /* AD reused as scratch */
            fr[j] = sqrt(orc_dot(AD, AD, n));
        }
        if (tr->final_residual_norms) {
            for (int j = 0; j < p0; ++j) tr->final_residual_norms[j] = NAN;
            for (int j = 0; j < p; ++j) tr->final_residual_norms[ids[j]] = fr[j];
        }
        double m = fr[0];
        for (int j = 0; j < p; ++j) m = (fr[j] < m) ? fr[j] : m; /* std::min_element */
        tr->final_minres = m;
    }
    free(X);
    free(R);
    free(D);
    free(Dn);
    free(AD);
    return rc;
}

int orc_ccg_solve(int n, int p, const double* A, const double* b, const double* X0,
                  const orc_opts* opts, orc_trace* tr) {
    return orc_block_solve(n, p, A, b, X0, opts, 0, tr);
}

int orc_mccg_solve(int n, int p, const double* A, const double* b, const double* X0,
                   const orc_opts* opts, orc_trace* tr) {
    return orc_block_solve(n, p, A, b, X0, opts, 1, tr);
}

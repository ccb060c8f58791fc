/*
 * gen_oracle.c -- CPU restatement of the BASELINE.json input generators.
 * TEST INFRASTRUCTURE ONLY (see ccg_oracle.c header).
 *
 * The reference has no generator for the BASELINE configs, so
 * DESIGN.md §3 defines them on top of the reference's counter-based
 * SplitMix64 streams (coopcg/rng.hpp:16-20 mix64, :35-39 next_u64,
 * :42-48 next_unit/next_uniform, :62-70 next_normal, :80-87 make_stream).
 * The product generates the same artifacts partly on the host and partly on
 * the GPU; tests compare both against this file bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ccg_oracle.h"

#define GOLDEN 0x9E3779B97F4A7C15ull
#define SID_RHS 3ull        /* rng.hpp StreamId::rhs */
#define SID_STARTS 4ull     /* rng.hpp StreamId::starts */
#define SID_DD_MATRIX 101ull
#define SID_HH_VECTORS 102ull

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t stream_key(uint64_t seed, uint64_t id, uint64_t extra) {
    return mix64(seed ^ mix64(id ^ mix64(extra)));
}
/* Draw number c (1-based, as Stream::next_u64 pre-increments its counter). */
static uint64_t draw(uint64_t key, uint64_t c) { return mix64(key + c * GOLDEN); }
static double unit53(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }
static double uniform_pm1(uint64_t key, uint64_t c) { return -1.0 + 2.0 * unit53(draw(key, c)); }
/* The t-th normal of a fresh stream: Box-Muller on draws 2t+1, 2t+2. */
static double normal_at(uint64_t key, uint64_t t) {
    double u1 = unit53(draw(key, 2 * t + 1));
    double u2 = unit53(draw(key, 2 * t + 2));
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double two_pi = 6.283185307179586476925286766559;
    return r * cos(two_pi * u2);
}

void orc_gen_diagdom(int n, uint64_t seed, double* A) {
    const uint64_t key = stream_key(seed, SID_DD_MATRIX, (uint64_t)n);
    const uint64_t un = (uint64_t)n;
    for (int i = 0; i < n; ++i) {
        A[(size_t)i * n + i] = 0.0;
        for (int j = i + 1; j < n; ++j) {
            const double u1 = uniform_pm1(key, (uint64_t)i * un + (uint64_t)j + 1);
            const double u2 = uniform_pm1(key, (uint64_t)j * un + (uint64_t)i + 1);
            const double a = (u1 + u2) * 0.5;
            A[(size_t)i * n + j] = a;
            A[(size_t)j * n + i] = a;
        }
    }
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j)
            if (j != i) acc += fabs(A[(size_t)i * n + j]);
        A[(size_t)i * n + i] = acc + 1.0;
    }
}

/* Rows [r0, r1) of the diagonally dominant A, row-major (r1 - r0) x n, each
 * element the same pure function of its index as orc_gen_diagdom (the pair
 * (min, max) draws the two uniforms; the diagonal is the ascending sum of the
 * row's |off-diagonal| values plus one).  Rows are independent, so the rows
 * run in parallel (OpenMP) with no change to any element's operation order:
 * this is how the full-size configs (n = 16384 .. 131072) are generated on
 * the host for the reference runs.  */
void orc_gen_diagdom_rows(int n, uint64_t seed, int r0, int r1, double* out) {
    const uint64_t key = stream_key(seed, SID_DD_MATRIX, (uint64_t)n);
    const uint64_t un = (uint64_t)n;
#pragma omp parallel for schedule(dynamic, 8)
    for (int i = r0; i < r1; ++i) {
        double* row = out + (size_t)(i - r0) * n;
        for (int j = 0; j < n; ++j) {
            if (j == i) continue;
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            const double u1 = uniform_pm1(key, (uint64_t)lo * un + (uint64_t)hi + 1);
            const double u2 = uniform_pm1(key, (uint64_t)hi * un + (uint64_t)lo + 1);
            row[j] = (u1 + u2) * 0.5;
        }
        double acc = 0.0;
        for (int j = 0; j < n; ++j)
            if (j != i) acc += fabs(row[j]);
        row[i] = acc + 1.0;
    }
}

void orc_gen_householder_factors(int n, int m, double kappa, uint64_t seed, double* V,
                                 double* lambda) {
    for (int i = 0; i < n; ++i) lambda[i] = pow(kappa, (double)i / (double)(n - 1));
    for (int r = 0; r < m; ++r) {
        const uint64_t key = stream_key(seed, SID_HH_VECTORS, (uint64_t)r);
        for (int i = 0; i < n; ++i) V[(size_t)r * n + i] = normal_at(key, (uint64_t)i);
    }
}

void orc_gen_householder(int n, int m, const double* V, const double* lambda, double* A) {
    memset(A, 0, sizeof(double) * (size_t)n * n);
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] = lambda[i];
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    for (int r = m - 1; r >= 0; --r) {
        const double* v = V + (size_t)r * n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) s += v[k] * v[k];
        for (int i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int k = 0; k < n; ++k) acc += A[(size_t)i * n + k] * v[k];
            w[i] = acc;
        }
        double c = 0.0;
        for (int i = 0; i < n; ++i) c += v[i] * w[i];
        const double t1 = 2.0 / s;
        const double t2 = (4.0 * c) / (s * s);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const double q = v[i] * w[j] + w[i] * v[j];
                const double m1 = A[(size_t)i * n + j] - t1 * q;
                A[(size_t)i * n + j] = m1 + t2 * (v[i] * v[j]);
            }
    }
    free(w);
}

/* orc_gen_householder with the row loops in parallel (OpenMP): every w_i is
 * still one sequential chain over k and every updated element the same
 * operation sequence, so the result is bit-identical for any thread count. */
void orc_gen_householder_par(int n, int m, const double* V, const double* lambda, double* A) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        memset(A + (size_t)i * n, 0, sizeof(double) * (size_t)n);
        A[(size_t)i * n + i] = lambda[i];
    }
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    for (int r = m - 1; r >= 0; --r) {
        const double* v = V + (size_t)r * n;
        double s = 0.0;
        for (int k = 0; k < n; ++k) s += v[k] * v[k];
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            double acc = 0.0;
            const double* row = A + (size_t)i * n;
            for (int k = 0; k < n; ++k) acc += row[k] * v[k];
            w[i] = acc;
        }
        double c = 0.0;
        for (int i = 0; i < n; ++i) c += v[i] * w[i];
        const double t1 = 2.0 / s;
        const double t2 = (4.0 * c) / (s * s);
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) {
            double* row = A + (size_t)i * n;
            const double vi = v[i], wi = w[i];
            for (int j = 0; j < n; ++j) {
                const double q = vi * w[j] + wi * v[j];
                const double m1 = row[j] - t1 * q;
                row[j] = m1 + t2 * (vi * v[j]);
            }
        }
    }
    free(w);
}

void orc_gen_rhs(int n, int kind, uint64_t seed, double* b) {
    const uint64_t key = stream_key(seed, SID_RHS, (uint64_t)n);
    for (int i = 0; i < n; ++i)
        b[i] = kind == 0 ? uniform_pm1(key, (uint64_t)i + 1) : normal_at(key, (uint64_t)i);
}

void orc_gen_starts(int n, int p, uint64_t seed, double* X0) {
    const uint64_t key = stream_key(seed, SID_STARTS, (uint64_t)n);
    for (int i = 0; i < n; ++i) X0[i] = 0.0;
    for (int j = 1; j < p; ++j)
        for (int i = 0; i < n; ++i)
            X0[(size_t)j * n + i] = uniform_pm1(key, (uint64_t)j * (uint64_t)n + (uint64_t)i + 1);
}

/*
 * jm_oracle.c — plain, slow, obviously-correct CPU ORACLE for the Eigen
 * benchmark update of ClangJIT (Finkel, Poliakoff, Richards, arXiv 1904.08555).
 *
 *   TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 *   bench.py's cpu_baseline / --impl reference legs may load this library.
 *   The product path (paper_1904_08555_b200/) never links, imports or calls
 *   it, and shares no code, header, constant or helper with it.
 *
 * What it computes (PAPER.md:362 prose; Listing 4; Listing 5
 * lines 406-408):
 *
 *     for r < repeat:   m = Ones + T(0.00005) * (m + (m*m))
 *
 * applied independently to each of `batch` n-by-n matrices, in the element
 * type T the caller names (float or double).  Readings
 * taken where the paper is silent:
 *   R1 (Q1) the addend is the listings' Matrix::Ones (all-ones J); the prose
 *           "I" (identity) is offered as addend=1.
 *   R2 (Q2) c = T(0.00005): the literal is rounded to T before use.
 *   R6 (Q6) the product sums k in ascending order with a separate multiply
 *           and add (this file is compiled with -ffp-contract=off, no
 *           -ffast-math, IEEE denormals).
 *   R7 (Q7) elementwise order: t = m + p; u = c*t; r = A + u  (as written).
 *   R8 (Q8) m*m is formed from the PRE-update m (Eigen evaluates products
 *           into a temporary), so the update is simultaneous.
 *   R5 (Q5) buffers are read as row-major m[i][j] = in[i*n + j]; reading them
 *           column-major gives the transposed result bitwise (O9), so both
 *           storage readings agree on the flat buffer.
 *   R9 (Q9) IEEE inf/NaN propagate; there is no convergence early exit.
 *
 * Pins (tests/test_oracle_pins.py): O1 SPEC.md:537 worked example, O3 the
 * hand-expanded n=2 step, O4/O5 closed-form fixed points, O6/O7/O8 invariant
 * families, O9 transpose equivariance, O10 exact rational brute force for
 * n=1..4, O11 R=0 / batch independence, O12 divergence for n>=35.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORACLE_F32 0
#define ORACLE_F64 1
#define ORACLE_ONES 0
#define ORACLE_IDENTITY 1

/* One update m -> r of one matrix, type double. */
static void step_f64(int n, int addend, const double *m, double *r) {
    const double c = (double)0.00005;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            double p = 0.0;
            for (int k = 0; k < n; ++k) {      /* (m*m)(i,j), ascending k */
                double prod = m[i * n + k] * m[k * n + j];
                p = p + prod;
            }
            double t = m[i * n + j] + p;        /* m + m*m */
            double u = c * t;                   /* T(0.00005) * (...) */
            /* Ones + u, or (prose reading) I + u */
            r[i * n + j] = (addend == ORACLE_ONES || i == j) ? 1.0 + u : u;
        }
    }
}

/* Same, type float: every operation rounds to float (T = float). */
static void step_f32(int n, int addend, const float *m, float *r) {
    const float c = (float)0.00005;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j) {
            float p = 0.0f;
            for (int k = 0; k < n; ++k) {
                float prod = m[i * n + k] * m[k * n + j];
                p = p + prod;
            }
            float t = m[i * n + j] + p;
            float u = c * t;
            r[i * n + j] = (addend == ORACLE_ONES || i == j) ? 1.0f + u : u;
        }
    }
}

typedef struct {
    int n, dtype, addend;
    int64_t b0, b1, repeat;
    const void *in;
    void *out;
} job_t;

static void *run_range(void *arg) {
    job_t *j = (job_t *)arg;
    const int n = j->n;
    const size_t nn = (size_t)n * (size_t)n;
    if (j->dtype == ORACLE_F64) {
        double *a = (double *)malloc(nn * sizeof(double));
        double *b = (double *)malloc(nn * sizeof(double));
        for (int64_t bi = j->b0; bi < j->b1; ++bi) {
            memcpy(a, (const double *)j->in + (size_t)bi * nn, nn * sizeof(double));
            for (int64_t r = 0; r < j->repeat; ++r) {
                step_f64(n, j->addend, a, b);
                double *t = a; a = b; b = t;    /* m = r */
            }
            memcpy((double *)j->out + (size_t)bi * nn, a, nn * sizeof(double));
        }
        free(a); free(b);
    } else {
        float *a = (float *)malloc(nn * sizeof(float));
        float *b = (float *)malloc(nn * sizeof(float));
        for (int64_t bi = j->b0; bi < j->b1; ++bi) {
            memcpy(a, (const float *)j->in + (size_t)bi * nn, nn * sizeof(float));
            for (int64_t r = 0; r < j->repeat; ++r) {
                step_f32(n, j->addend, a, b);
                float *t = a; a = b; b = t;
            }
            memcpy((float *)j->out + (size_t)bi * nn, a, nn * sizeof(float));
        }
        free(a); free(b);
    }
    return NULL;
}

/*
 * Batched small matrix multiply-accumulate — the RAJA benchmark of PAPER.md
 * §5.1, Listing 8 (lines 562-600):
 *     out_matrix[MAT2D(i,j,size)] += input_matrix1[MAT2D(i,k,size)] *
 *                                    input_matrix2[MAT2D(k,j,size)]
 * over the loop nest (matrices, i, j, k), innermost k ascending, one multiply
 * and one add per iteration (separate roundings).  Reading R16:
 * the listing's lambda ignores the `matrices` index, so as printed every batch
 * entry accumulates into ONE output; the batch form c[b] += a[b] * b[b] (each
 * entry its own three matrices) is the evident intent and is what this
 * computes.  Row-major MAT2D(r,c,size) = r*size + c, as in the listing.
 */
static void *mm_range(void *arg) {
    job_t *j = (job_t *)arg;
    const int n = j->n;
    const size_t nn = (size_t)n * (size_t)n;
    const void *const *ab = (const void *const *)j->in;   /* {a, b} */
    for (int64_t bi = j->b0; bi < j->b1; ++bi) {
        if (j->dtype == ORACLE_F64) {
            const double *a = (const double *)ab[0] + (size_t)bi * nn;
            const double *b = (const double *)ab[1] + (size_t)bi * nn;
            double *c = (double *)j->out + (size_t)bi * nn;
            for (int i = 0; i < n; ++i)
                for (int jj = 0; jj < n; ++jj)
                    for (int k = 0; k < n; ++k) {
                        double prod = a[i * n + k] * b[k * n + jj];
                        c[i * n + jj] = c[i * n + jj] + prod;
                    }
        } else {
            const float *a = (const float *)ab[0] + (size_t)bi * nn;
            const float *b = (const float *)ab[1] + (size_t)bi * nn;
            float *c = (float *)j->out + (size_t)bi * nn;
            for (int i = 0; i < n; ++i)
                for (int jj = 0; jj < n; ++jj)
                    for (int k = 0; k < n; ++k) {
                        float prod = a[i * n + k] * b[k * n + jj];
                        c[i * n + jj] = c[i * n + jj] + prod;
                    }
        }
    }
    return NULL;
}

/* c[b] += a[b] * b[b] for b in [0, batch) (host buffers, c updated in place). */
int jm_oracle_matmul(int n, int dtype, int64_t batch, const void *a, const void *b, void *c,
                     int threads) {
    if (n < 1 || batch < 0) return -1;
    if (dtype != ORACLE_F32 && dtype != ORACLE_F64) return -1;
    if (batch == 0) return 0;
    if (threads < 1) threads = 1;
    if ((int64_t)threads > batch) threads = (int)batch;
    const void *ab[2] = {a, b};
    job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].n = n; jobs[t].dtype = dtype; jobs[t].addend = 0;
        jobs[t].b0 = batch * t / threads;
        jobs[t].b1 = batch * (t + 1) / threads;
        jobs[t].repeat = 0; jobs[t].in = ab; jobs[t].out = c;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, mm_range, &jobs[t]);
    mm_range(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs); free(tids);
    return 0;
}

/*
 * Laghos 2D mass-operator action, rMassMultAdd2D<NUM_DOFS_1D, NUM_QUAD_1D>
 * (§5.3, Listing 12: the kernel whose ~32 explicit
 * instantiations ClangJIT replaces; Fig. 7 lines 765-785 time it on 10,000
 * elements).  The paper names the kernel but does not print it; reading R18
 * takes the standard sum-factorised partial-assembly mass action
 * of Laghos/MFEM, with D = NUM_DOFS_1D, Q = NUM_QUAD_1D, for each element e:
 *     S[qy][qx] = sum_dy sum_dx B[qy][dy] B[qx][dx] X[e][dy][dx]   (x to quad points)
 *     S[qy][qx] *= op[e][qy][qx]                                    (quadrature weights)
 *     Y[e][dy][dx] += sum_qy sum_qx B[qy][dy] B[qx][dx] S[qy][qx]   (back to dofs)
 * evaluated in Laghos' loop order: first contract dx, then dy (and qx, then
 * qy on the way back), ascending indices, separate multiply and add.  Layouts
 * (row-major here): B is Q x D (B[q*D + d], Laghos' dofToQuad), op is E x Q x Q
 * (op[e*Q*Q + qy*Q + qx]), x and y are E x D x D (x[e*D*D + dy*D + dx]); the
 * transposed basis (quadToDof) is B^T.  y is updated in place.
 */
typedef struct {
    int D, Q;
    int64_t e0, e1;
    const double *B, *op, *x;
    double *y;
} mass_job_t;

static void *mass_range(void *arg) {
    mass_job_t *j = (mass_job_t *)arg;
    const int D = j->D, Q = j->Q;
    double *sol_xy = (double *)malloc((size_t)Q * Q * sizeof(double));
    double *sol_x = (double *)malloc((size_t)(Q > D ? Q : D) * sizeof(double));
    for (int64_t e = j->e0; e < j->e1; ++e) {
        const double *x = j->x + (size_t)e * D * D;
        const double *op = j->op + (size_t)e * Q * Q;
        double *y = j->y + (size_t)e * D * D;
        for (int i = 0; i < Q * Q; ++i) sol_xy[i] = 0.0;
        for (int dy = 0; dy < D; ++dy) {
            for (int qx = 0; qx < Q; ++qx) sol_x[qx] = 0.0;
            for (int dx = 0; dx < D; ++dx) {
                const double s = x[dy * D + dx];
                for (int qx = 0; qx < Q; ++qx) sol_x[qx] = sol_x[qx] + j->B[qx * D + dx] * s;
            }
            for (int qy = 0; qy < Q; ++qy) {
                const double d2q = j->B[qy * D + dy];
                for (int qx = 0; qx < Q; ++qx) sol_xy[qy * Q + qx] = sol_xy[qy * Q + qx] + d2q * sol_x[qx];
            }
        }
        for (int qy = 0; qy < Q; ++qy)
            for (int qx = 0; qx < Q; ++qx) sol_xy[qy * Q + qx] = sol_xy[qy * Q + qx] * op[qy * Q + qx];
        for (int qy = 0; qy < Q; ++qy) {
            for (int dx = 0; dx < D; ++dx) sol_x[dx] = 0.0;
            for (int qx = 0; qx < Q; ++qx) {
                const double s = sol_xy[qy * Q + qx];
                for (int dx = 0; dx < D; ++dx) sol_x[dx] = sol_x[dx] + j->B[qx * D + dx] * s;
            }
            for (int dy = 0; dy < D; ++dy) {
                const double q2d = j->B[qy * D + dy];
                for (int dx = 0; dx < D; ++dx) y[dy * D + dx] = y[dy * D + dx] + q2d * sol_x[dx];
            }
        }
    }
    free(sol_xy);
    free(sol_x);
    return NULL;
}

int jm_oracle_mass(int D, int Q, int64_t elements, const double *B, const double *op, const double *x,
                   double *y, int threads) {
    if (D < 1 || Q < 1 || elements < 0) return -1;
    if (elements == 0) return 0;
    if (threads < 1) threads = 1;
    if ((int64_t)threads > elements) threads = (int)elements;
    mass_job_t *jobs = (mass_job_t *)calloc((size_t)threads, sizeof(mass_job_t));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].D = D; jobs[t].Q = Q;
        jobs[t].e0 = elements * t / threads;
        jobs[t].e1 = elements * (t + 1) / threads;
        jobs[t].B = B; jobs[t].op = op; jobs[t].x = x; jobs[t].y = y;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, mass_range, &jobs[t]);
    mass_range(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs); free(tids);
    return 0;
}

/*
 * out[b] = f^repeat(in[b]) for b in [0, batch).  `in` and `out` are host
 * buffers of batch*n*n elements of the named type; they may be the same
 * buffer.  threads <= 0 means 1.  Returns 0, or -1 on bad arguments.
 */
int jm_oracle_run(int n, int dtype, int addend, int64_t batch, int64_t repeat,
                  const void *in, void *out, int threads) {
    if (n < 1 || batch < 0 || repeat < 0) return -1;
    if (dtype != ORACLE_F32 && dtype != ORACLE_F64) return -1;
    if (addend != ORACLE_ONES && addend != ORACLE_IDENTITY) return -1;
    if (batch == 0) return 0;
    if (threads < 1) threads = 1;
    if ((int64_t)threads > batch) threads = (int)batch;
    job_t *jobs = (job_t *)calloc((size_t)threads, sizeof(job_t));
    pthread_t *tids = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].n = n; jobs[t].dtype = dtype; jobs[t].addend = addend;
        jobs[t].b0 = batch * t / threads;
        jobs[t].b1 = batch * (t + 1) / threads;
        jobs[t].repeat = repeat; jobs[t].in = in; jobs[t].out = out;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tids[t], NULL, run_range, &jobs[t]);
    run_range(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs); free(tids);
    return 0;
}

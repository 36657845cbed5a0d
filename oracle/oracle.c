/*
 * oracle.c -- CPU ORACLE for the single-scan min-sum LDPC decoder.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_cs_0609090_b200/);
 * its inputs come from ldpcgen/ or from the tests themselves.
 *
 * Plain, slow, obviously-correct C following X. Huang, "Single-Scan Min-Sum
 * Algorithms for Fast Decoding of LDPC Codes":
 *   ENG_TWOSCAN_NAIVE  §3 Eq.(1)/(2) literally (O(dc^2) check rule): the plain
 *                      definition that the single-scan forms equal.
 *   ENG_TWOSCAN        §3 with the two-minima check rule (P:255-292 observation).
 *   ENG_SINGLESCAN     §4 Eq.(3) block with per-edge L_mn storage.
 *   ENG_COMPACT        §5 memory-efficient single-scan (variants P:338-353):
 *                      the CUDA path's direct parity target.
 *   ENG_LAYERED_FULL   the Eq.(3) block with a single in-place posterior array (the
 *                      layered / Gauss-Seidel reading, DESIGN D25),
 *                      per-edge L_mn and Eq.(1) evaluated literally.
 *   ENG_LAYERED        the same schedule over the §5 compact state (GPU layered target).
 * Numeric types: int32 (fixed point, offset + clamp), double, float (one rounding per
 * operation, D11; posterior sums exact and rounded once, D28).
 * Readings of silent/ambiguous passages are listed in DESIGN.md §3 (D1-D27).
 * Parity pins: tests/test_oracle.py, tests/golden/ (none of this file is "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

enum { ENG_TWOSCAN_NAIVE = 0, ENG_TWOSCAN = 1, ENG_SINGLESCAN = 2, ENG_COMPACT = 3,
       ENG_LAYERED_FULL = 4, ENG_LAYERED = 5 };

typedef struct {
    int32_t max_iter;     /* K >= 1 */
    int32_t early_stop;   /* stop when H x̂ = 0, checked at k = 0 too (D10) */
    int32_t beta_i;       /* int: offset beta in LSBs */
    int32_t clamp_i;      /* int: magnitude clamp Q (0 = none) */
    double alpha;         /* float: normalization lambda (1 = none) */
    double beta_f;        /* float: offset beta (0 = none) */
    /* optional per-iteration schedules (NULL = the constants above), K entries:
     * lambda_k and beta_k of PAPER.md P:179 */
    const int32_t *beta_i_sched;
    const double *alpha_sched;
    const double *beta_f_sched;
} orc_params;

typedef struct {
    int N, M;
    const int32_t *row_ptr, *col_idx;  /* N(m): check -> variable addressing */
    int32_t *vptr, *vedge;             /* M(n): variable -> check addressing (two-scan only) */
} orc_code;

static int orc_code_init(orc_code *c, int N, int M, const int32_t *row_ptr, const int32_t *col_idx) {
    c->N = N; c->M = M; c->row_ptr = row_ptr; c->col_idx = col_idx;
    int64_t E = row_ptr[M];
    c->vptr = calloc((size_t)N + 1, sizeof(int32_t));
    c->vedge = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
    for (int64_t e = 0; e < E; ++e) {
        if (col_idx[e] < 0 || col_idx[e] >= N) return -1;
        c->vptr[col_idx[e] + 1]++;
    }
    for (int n = 0; n < N; ++n) c->vptr[n + 1] += c->vptr[n];
    int32_t *fill = malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    memcpy(fill, c->vptr, sizeof(int32_t) * (size_t)N);
    /* rows visited in ascending m, so each M(n) list is in ascending m */
    for (int m = 0; m < M; ++m)
        for (int32_t e = row_ptr[m]; e < row_ptr[m + 1]; ++e) c->vedge[fill[col_idx[e]]++] = e;
    free(fill);
    return 0;
}
static void orc_code_free(orc_code *c) { free(c->vptr); free(c->vedge); }

#define FN2(a, b) a##_##b
#define FN1(a, b) FN2(a, b)

/* Sums of several messages into a posterior (the flooding Z^(k)_n = Z^(0)_n + sum_m L_mn of
 * P:164-165 / P:318-322 and the two-scan variable rule Eq.(2)) go through an
 * accumulator type ACC: ACC_OF(x) enters a value, VAL_OF(a) leaves.  int and f64: the value
 * type itself, added in ascending m.  f32 (reading D28): the sum is evaluated
 * EXACTLY and rounded to fp32 once -- every term is placed on the fixed-point grid 2^-34
 * (exact for |x| >= 2^-11, round-half-even below), the grid integers are added in int64 (no
 * overflow: |x| <= 2^20 by the saturation below and at most 255 terms), and the total is
 * rounded to the nearest fp32.  Integer addition is associative, so the result does not
 * depend on the order of the terms. */
#define ORC_F32_GRID 34
#define ORC_F32_SAT 1048576.0f   /* 2^20: fp32 channel LLRs and message magnitudes saturate here (D28) */
static inline int64_t orc_f32_to_grid(float x) { return (int64_t)nearbyint(ldexp((double)x, ORC_F32_GRID)); }
static inline float orc_grid_to_f32(int64_t a) { return ldexpf((float)a, -ORC_F32_GRID); }

/* fixed point: raw integer LSB units */
#define VAL int32_t
#define VAL_IS_INT 1
#define VAL_IS_F32 0
#define ACC int32_t
#define ACC_OF(x) (x)
#define VAL_OF(a) (a)
#define FN(x) FN1(x, i32)
#include "engine.inc"
#undef VAL
#undef VAL_IS_INT
#undef VAL_IS_F32
#undef ACC
#undef ACC_OF
#undef VAL_OF
#undef FN

/* float64 */
#define VAL double
#define VAL_IS_INT 0
#define VAL_IS_F32 0
#define ACC double
#define ACC_OF(x) (x)
#define VAL_OF(a) (a)
#define FN(x) FN1(x, f64)
#include "engine.inc"
#undef VAL
#undef VAL_IS_INT
#undef VAL_IS_F32
#undef ACC
#undef ACC_OF
#undef VAL_OF
#undef FN

/* float32 (reading D11: one round-to-nearest per operation, no contraction; reading D28:
 * posterior sums exact, rounded once) */
#define VAL float
#define VAL_IS_INT 0
#define VAL_IS_F32 1
#define ACC int64_t
#define ACC_OF(x) orc_f32_to_grid(x)
#define VAL_OF(a) orc_grid_to_f32(a)
#define FN(x) FN1(x, f32)
#include "engine.inc"
#undef VAL
#undef VAL_IS_INT
#undef VAL_IS_F32
#undef ACC
#undef ACC_OF
#undef VAL_OF
#undef FN

/* test hooks for the D28 accumulator (tests/test_oracle.py pins it against exact rational sums) */
float orc_f32_exact_sum(int n, const float *x) {
    int64_t a = 0;
    for (int i = 0; i < n; ++i) a += orc_f32_to_grid(x[i] > ORC_F32_SAT ? ORC_F32_SAT : (x[i] < -ORC_F32_SAT ? -ORC_F32_SAT : x[i]));
    return orc_grid_to_f32(a);
}

int orc_hardware_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

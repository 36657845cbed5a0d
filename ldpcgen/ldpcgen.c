/*
 * ldpcgen.c -- seeded synthetic INPUT generators for the LDPC decoder tests and bench.
 *
 * This module holds none of the decoding method's arithmetic: it only builds
 * parity-check matrices (H in CSR, optional QC shift table) and channel LLRs.
 * Both the CPU oracle (oracle/) and the CUDA path (paper_cs_0609090_b200/)
 * consume its outputs; neither shares any other code.
 *
 * Constructions follow SURVEY.md §8(c) D18-D21 / §8(d) (the paper's own
 * workloads -- China-DTMB QC codes, DVB-S2 codes, MacKay codes
 * (§1) -- are not available; these synthetic codes stand in with the same shapes).
 *
 * Channel: BPSK over AWGN, y = (-1)^x + xi, all-zero codeword, Z0 = 2y/sigma^2
 * (§2).  Counter-based generator so any frame range can be
 * regenerated independently (SURVEY.md §8(d) "Generator").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

/* ---------------------------------------------------------------- RNG */
static inline uint64_t sm_final(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t splitmix64(uint64_t x) { return sm_final(x + 0x9E3779B97F4A7C15ULL); }

typedef struct { uint64_t s; } rng_t;
static inline uint64_t rng_next(rng_t *r) { r->s += 0x9E3779B97F4A7C15ULL; return sm_final(r->s); }
/* uniform integer in [0, n) */
static inline uint64_t rng_below(rng_t *r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}
static void shuffle_i32(rng_t *r, int32_t *a, int64_t n) {
    for (int64_t i = n - 1; i > 0; --i) {
        int64_t j = (int64_t)rng_below(r, (uint64_t)i + 1);
        int32_t t = a[i]; a[i] = a[j]; a[j] = t;
    }
}

uint64_t lg_splitmix64(uint64_t x) { return splitmix64(x); }

/* ------------------------------------------------------- edge-list utils */
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Build CSR (rows = checks) from an edge list (chk[e], var[e]); columns sorted.
 * row_ptr must have M+1 entries, col_idx E entries. Returns 0, or -1 on duplicates. */
static int edges_to_csr(int M, int64_t E, const int32_t *chk, const int32_t *var,
                        int32_t *row_ptr, int32_t *col_idx) {
    memset(row_ptr, 0, sizeof(int32_t) * (size_t)(M + 1));
    for (int64_t e = 0; e < E; ++e) row_ptr[chk[e] + 1]++;
    for (int m = 0; m < M; ++m) row_ptr[m + 1] += row_ptr[m];
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)M);
    for (int m = 0; m < M; ++m) fill[m] = row_ptr[m];
    for (int64_t e = 0; e < E; ++e) col_idx[fill[chk[e]]++] = var[e];
    free(fill);
    int dup = 0;
    for (int m = 0; m < M; ++m) {
        qsort(col_idx + row_ptr[m], (size_t)(row_ptr[m + 1] - row_ptr[m]), sizeof(int32_t), cmp_i32);
        for (int32_t k = row_ptr[m] + 1; k < row_ptr[m + 1]; ++k)
            if (col_idx[k] == col_idx[k - 1]) dup = 1;
    }
    return dup ? -1 : 0;
}

/* ------------------------------------------- (dv,dc)-regular random code
 * Socket (configuration-model) construction; duplicates and (optionally)
 * 4-cycles are removed by LOCAL re-draw: the check endpoint of an offending
 * edge is swapped with that of a uniformly random other edge (degrees are
 * preserved), repeated until clean.
 * Returns number of repair rounds (>=0) or -1 on failure. */
int lg_regular(int N, int dv, int dc, uint64_t seed, int remove_4cycles,
               int32_t *row_ptr /* M+1 */, int32_t *col_idx /* N*dv */) {
    if (N <= 0 || dv <= 0 || dc <= 1 || (N * dv) % dc) return -1;
    int M = N * dv / dc;
    int64_t E = (int64_t)N * dv;
    rng_t r = { splitmix64(seed ^ 0x5EEDC0DEULL) };
    int32_t *var = malloc(sizeof(int32_t) * E), *chk = malloc(sizeof(int32_t) * E);
    for (int64_t e = 0; e < E; ++e) { var[e] = (int32_t)(e / dv); chk[e] = (int32_t)(e / dc); }
    shuffle_i32(&r, chk, E);
    int32_t *bad = malloc(sizeof(int32_t) * E);
    int32_t *vstart = malloc(sizeof(int32_t) * (N + 1));
    int32_t *vchk = malloc(sizeof(int32_t) * E);
    int32_t *vedge = malloc(sizeof(int32_t) * E);
    /* pair table for 4-cycle detection: hash of (m1,m2) -> first variable seen */
    int64_t HS = 1; while (HS < E * 8) HS <<= 1;
    uint64_t *hkey = malloc(sizeof(uint64_t) * HS);
    int32_t *hval = malloc(sizeof(int32_t) * HS);
    int rounds = 0;
    for (; rounds < 100000; ++rounds) {
        /* var-major view */
        memset(vstart, 0, sizeof(int32_t) * (N + 1));
        for (int64_t e = 0; e < E; ++e) vstart[var[e] + 1]++;
        for (int n = 0; n < N; ++n) vstart[n + 1] += vstart[n];
        {
            int32_t *f = malloc(sizeof(int32_t) * N);
            memcpy(f, vstart, sizeof(int32_t) * N);
            for (int64_t e = 0; e < E; ++e) { vchk[f[var[e]]] = chk[e]; vedge[f[var[e]]++] = (int32_t)e; }
            free(f);
        }
        int64_t nbad = 0;
        /* duplicates */
        for (int n = 0; n < N; ++n)
            for (int32_t a = vstart[n]; a < vstart[n + 1]; ++a)
                for (int32_t b = a + 1; b < vstart[n + 1]; ++b)
                    if (vchk[a] == vchk[b]) bad[nbad++] = vedge[b];
        if (remove_4cycles) {
            for (int64_t h = 0; h < HS; ++h) hkey[h] = ~0ULL;
            for (int n = 0; n < N; ++n)
                for (int32_t a = vstart[n]; a < vstart[n + 1]; ++a)
                    for (int32_t b = vstart[n]; b < vstart[n + 1]; ++b) {
                        int32_t m1 = vchk[a], m2 = vchk[b];
                        if (m1 >= m2) continue;
                        uint64_t key = ((uint64_t)(uint32_t)m1 << 32) | (uint32_t)m2;
                        uint64_t h = splitmix64(key) & (uint64_t)(HS - 1);
                        while (hkey[h] != ~0ULL && hkey[h] != key) h = (h + 1) & (uint64_t)(HS - 1);
                        if (hkey[h] == ~0ULL) { hkey[h] = key; hval[h] = n; }
                        else if (hval[h] != n) bad[nbad++] = vedge[a];  /* second variable shares (m1,m2) */
                    }
        }
        if (nbad == 0) break;
        for (int64_t i = 0; i < nbad; ++i) {
            int64_t e = bad[i], f = (int64_t)rng_below(&r, (uint64_t)E);
            int32_t t = chk[e]; chk[e] = chk[f]; chk[f] = t;
        }
    }
    int ok = (rounds < 100000) && edges_to_csr(M, E, chk, var, row_ptr, col_idx) == 0;
    free(var); free(chk); free(bad); free(vstart); free(vchk); free(vedge); free(hkey); free(hval);
    return ok ? rounds : -1;
}

/* ------------------------------------------------ QC code (DTMB shape)
 * Base matrix mb x nb, circulant size Z.  col_w[j] is the weight of base column j;
 * row weights are balanced (differ by at most one).  Base entries (i,j) get a
 * uniform shift in [0,Z); entry s puts a 1 at (i*Z + r, j*Z + (r+s) mod Z).
 * No duplicate base entries; 4-cycles are NOT removed.
 * shifts: mb*nb int16, -1 = empty.  Returns 0 or -1. */
int lg_qc_base(int mb, int nb, int Z, const int32_t *col_w, uint64_t seed, int16_t *shifts) {
    int64_t E = 0;
    for (int j = 0; j < nb; ++j) { if (col_w[j] < 0 || col_w[j] > mb) return -1; E += col_w[j]; }
    rng_t r = { splitmix64(seed ^ 0x0C0C0C0CULL) };
    int32_t *var = malloc(sizeof(int32_t) * E), *chk = malloc(sizeof(int32_t) * E);
    int64_t e = 0;
    for (int j = 0; j < nb; ++j) for (int k = 0; k < col_w[j]; ++k) var[e++] = j;
    /* balanced row sockets */
    for (e = 0; e < E; ++e) chk[e] = (int32_t)(e % mb);
    shuffle_i32(&r, chk, E);
    int rounds;
    for (rounds = 0; rounds < 100000; ++rounds) {
        /* find duplicate (i,j) */
        int64_t nbad = 0;
        char *seen = calloc((size_t)mb * nb, 1);
        int32_t *bad = malloc(sizeof(int32_t) * E);
        for (e = 0; e < E; ++e) {
            size_t k = (size_t)chk[e] * nb + var[e];
            if (seen[k]) bad[nbad++] = (int32_t)e; else seen[k] = 1;
        }
        free(seen);
        for (int64_t i = 0; i < nbad; ++i) {
            int64_t a = bad[i], b = (int64_t)rng_below(&r, (uint64_t)E);
            int32_t t = chk[a]; chk[a] = chk[b]; chk[b] = t;
        }
        free(bad);
        if (nbad == 0) break;
    }
    if (rounds >= 100000) { free(var); free(chk); return -1; }
    for (int64_t k = 0; k < (int64_t)mb * nb; ++k) shifts[k] = -1;
    /* shifts drawn in (row, col) order so the table is independent of socket order */
    for (int i = 0; i < mb; ++i) for (int j = 0; j < nb; ++j) {
        int present = 0;
        for (e = 0; e < E; ++e) if (chk[e] == i && var[e] == j) { present = 1; break; }
        if (present) shifts[(size_t)i * nb + j] = (int16_t)rng_below(&r, (uint64_t)Z);
    }
    free(var); free(chk);
    return 0;
}

/* Expand a QC base shift table into CSR (columns sorted). */
int lg_qc_expand(int mb, int nb, int Z, const int16_t *shifts, int32_t *row_ptr, int32_t *col_idx) {
    int32_t k = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < mb; ++i)
        for (int r = 0; r < Z; ++r) {
            int32_t start = k;
            for (int j = 0; j < nb; ++j) {
                int s = shifts[(size_t)i * nb + j];
                if (s < 0) continue;
                col_idx[k++] = j * Z + (r + s) % Z;
            }
            qsort(col_idx + start, (size_t)(k - start), sizeof(int32_t), cmp_i32);
            row_ptr[i * Z + r + 1] = k;
        }
    return 0;
}

/* ------------------------------------- DVB-S2-shaped irregular code
 * N = K + M variables.  Info columns 0..n_hi-1 have weight w_hi, columns
 * n_hi..K-1 weight w_lo; info edges are socket-balanced over the checks
 * (each check gets exactly (n_hi*w_hi + (K-n_hi)*w_lo)/M info edges),
 * duplicates repaired by swaps.  Parity columns form the dual-diagonal
 * staircase: column K+p covers rows p and p+1 (the last column covers row
 * M-1 only).  (SURVEY.md §8(c) D19.)  Returns 0 or -1. */
int lg_dvbs2like(int N, int M, int n_hi, int w_hi, int w_lo, uint64_t seed,
                 int32_t *row_ptr, int32_t *col_idx) {
    int K = N - M;
    if (K <= 0 || n_hi > K) return -1;
    int64_t Ei = (int64_t)n_hi * w_hi + (int64_t)(K - n_hi) * w_lo;
    if (Ei % M) return -1;
    int64_t E = Ei + 2LL * M - 1;
    rng_t r = { splitmix64(seed ^ 0xD5B52ULL) };
    int32_t *var = malloc(sizeof(int32_t) * E), *chk = malloc(sizeof(int32_t) * E);
    int64_t e = 0;
    for (int j = 0; j < K; ++j) { int w = j < n_hi ? w_hi : w_lo; for (int k = 0; k < w; ++k) var[e++] = j; }
    for (e = 0; e < Ei; ++e) chk[e] = (int32_t)(e % M);
    shuffle_i32(&r, chk, Ei);
    int rounds;
    for (rounds = 0; rounds < 100000; ++rounds) {
        int64_t nbad = 0;
        /* duplicates among info edges: per variable, its checks must be distinct */
        int32_t *bad = malloc(sizeof(int32_t) * Ei);
        int64_t e0 = 0;
        for (int j = 0; j < K; ++j) {
            int w = j < n_hi ? w_hi : w_lo;
            for (int a = 0; a < w; ++a) for (int b = a + 1; b < w; ++b)
                if (chk[e0 + a] == chk[e0 + b]) { bad[nbad++] = (int32_t)(e0 + b); }
            e0 += w;
        }
        for (int64_t i = 0; i < nbad; ++i) {
            int64_t a = bad[i], b = (int64_t)rng_below(&r, (uint64_t)Ei);
            int32_t t = chk[a]; chk[a] = chk[b]; chk[b] = t;
        }
        free(bad);
        if (nbad == 0) break;
    }
    if (rounds >= 100000) { free(var); free(chk); return -1; }
    e = Ei;
    for (int p = 0; p < M; ++p) {
        var[e] = K + p; chk[e] = p; ++e;
        if (p + 1 < M) { var[e] = K + p; chk[e] = p + 1; ++e; }
    }
    int rc = edges_to_csr(M, E, chk, var, row_ptr, col_idx);
    free(var); free(chk);
    return rc;
}

/* --------------------------------------------------------- channel LLRs
 * For global frame f and position n: pair i = n/2, h1 = splitmix64(key + 2c),
 * h2 = splitmix64(key + 2c + 1), c = f*2^32 + i, key = splitmix64(noise_seed);
 * u1 = ((h1>>11)+1) 2^-53, u2 = (h2>>11) 2^-53; Box-Muller in double gives
 * g_{2i} = sqrt(-2 ln u1) cos(2 pi u2), g_{2i+1} = ... sin(...).
 * y = 1 + sigma g (all-zero codeword, BPSK +1); Z0 = 2y/sigma^2.
 * sigma2 == 0 gives noiseless y = 1 and Z0 = 2 (scaled mode is undefined there,
 * so noiseless frames use Z0 = y scaled by 2, i.e. 2.0). */
static void llr_frame_double(uint64_t key, int64_t f, int N, double sigma2, double *out) {
    double sigma = sqrt(sigma2);
    double scale = sigma2 > 0 ? 2.0 / sigma2 : 2.0;
    for (int i = 0; 2 * i < N; ++i) {
        uint64_t c = ((uint64_t)f << 32) + (uint64_t)i;
        uint64_t h1 = splitmix64(key + 2 * c), h2 = splitmix64(key + 2 * c + 1);
        double u1 = (double)((h1 >> 11) + 1) * 0x1.0p-53;
        double u2 = (double)(h2 >> 11) * 0x1.0p-53;
        double rad = sqrt(-2.0 * log(u1));
        double g0 = rad * cos(2.0 * M_PI * u2), g1 = rad * sin(2.0 * M_PI * u2);
        out[2 * i] = scale * (1.0 + sigma * g0);
        if (2 * i + 1 < N) out[2 * i + 1] = scale * (1.0 + sigma * g1);
    }
}

/* kind: 0 = float64, 1 = float32, 2 = int16 quantized, 3 = int8 quantized */
typedef struct {
    uint64_t key; int64_t f0; int64_t nf; int N; double sigma2;
    int kind; int frac_bits; int clamp; void *out;
    int64_t lo, hi;
} llr_job;

static void *llr_worker(void *arg) {
    llr_job *j = (llr_job *)arg;
    double *buf = malloc(sizeof(double) * (size_t)j->N);
    double q = ldexp(1.0, j->frac_bits);
    for (int64_t t = j->lo; t < j->hi; ++t) {
        llr_frame_double(j->key, j->f0 + t, j->N, j->sigma2, buf);
        size_t base = (size_t)t * (size_t)j->N;
        for (int n = 0; n < j->N; ++n) {
            double v = buf[n];
            switch (j->kind) {
            case 0: ((double *)j->out)[base + n] = v == 0.0 ? 0.0 : v; break;
            case 1: { float x = (float)v; if (x == 0.0f) x = 0.0f; ((float *)j->out)[base + n] = x; break; }
            default: {
                /* D12: round-half-even of LLR*2^f in double, symmetric clamp +-Q */
                double x = rint(v * q);
                if (x > j->clamp) x = j->clamp;
                if (x < -j->clamp) x = -j->clamp;
                if (j->kind == 2) ((int16_t *)j->out)[base + n] = (int16_t)x;
                else ((int8_t *)j->out)[base + n] = (int8_t)x;
            }
            }
        }
    }
    free(buf);
    return NULL;
}

/* Generate LLRs for frames [f0, f0+nf) into out ([nf][N], row-major). */
int lg_llr(uint64_t noise_seed, int64_t f0, int64_t nf, int N, double sigma2,
           int kind, int frac_bits, int clamp, void *out, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nf < nthreads) nthreads = (int)(nf > 0 ? nf : 1);
    pthread_t th[256];
    llr_job jobs[256];
    uint64_t key = splitmix64(noise_seed);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (llr_job){ key, f0, nf, N, sigma2, kind, frac_bits, clamp, out,
                             nf * t / nthreads, nf * (t + 1) / nthreads };
        pthread_create(&th[t], NULL, llr_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* one standard-normal pair for (noise_seed, f, i) -- exposed for statistical tests */
void lg_gauss_pair(uint64_t noise_seed, int64_t f, int64_t i, double *g0, double *g1) {
    uint64_t key = splitmix64(noise_seed);
    uint64_t c = ((uint64_t)f << 32) + (uint64_t)i;
    uint64_t h1 = splitmix64(key + 2 * c), h2 = splitmix64(key + 2 * c + 1);
    double u1 = (double)((h1 >> 11) + 1) * 0x1.0p-53;
    double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    double rad = sqrt(-2.0 * log(u1));
    *g0 = rad * cos(2.0 * M_PI * u2);
    *g1 = rad * sin(2.0 * M_PI * u2);
}

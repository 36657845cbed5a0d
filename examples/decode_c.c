/*
 * decode_c.c -- using libldpc.so from plain C (no Python, no PyTorch): the C ABI of
 * include/ldpc.h end to end.
 *
 * Builds a small quasi-cyclic code (3 x 6 base matrix, Z = 16: N = 96, M = 48) from its
 * shift table, decodes a few all-zero-codeword frames with both entry points (device
 * buffers via ldpc_decode_batch, host buffers via ldpc_decode_batch_host), and checks
 * what the decoder must do on them: a frame of confident LLRs stops at iteration 0
 * (early stop), frames with one or two unreliable wrong-sign LLRs are corrected to
 * the all-zero codeword, and both entry points give identical outputs.  Exit status 0 on
 * success.
 *
 *   make examples/decode_c && examples/decode_c
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "ldpc.h"

#define MB 3
#define NB 6
#define Z 16
#define N (NB * Z)
#define M (MB * Z)
#define F 4

static int fails = 0;
#define CHECK(cond, ...)                      \
    do {                                      \
        if (!(cond)) {                        \
            fprintf(stderr, "FAIL: " __VA_ARGS__); \
            fputc('\n', stderr);              \
            ++fails;                          \
        }                                     \
    } while (0)
#define LDPC(call)                                                                                      \
    do {                                                                                                \
        ldpc_status s_ = (call);                                                                        \
        if (s_ != LDPC_OK) {                                                                            \
            fprintf(stderr, "%s: %s (%s)\n", #call, ldpc_status_string(s_), ldpc_last_error_detail()); \
            return 1;                                                                                   \
        }                                                                                               \
    } while (0)
#define CUDA(call)                                                                  \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));             \
            return 1;                                                               \
        }                                                                           \
    } while (0)

int main(void) {
    /* base matrix: every entry present (column degree 3, row degree 6), distinct shifts */
    static const int16_t shift[MB * NB] = {0, 1, 2, 3, 5, 8,
                                           0, 3, 6, 9, 12, 15,
                                           0, 7, 13, 2, 10, 4};
    int32_t row_ptr[M + 1], col_idx[M * NB];
    int e = 0;
    for (int i = 0; i < MB; ++i)
        for (int r = 0; r < Z; ++r) {
            row_ptr[i * Z + r] = e;
            for (int j = 0; j < NB; ++j) col_idx[e++] = j * Z + (r + shift[i * NB + j]) % Z;   /* ascending j */
        }
    row_ptr[M] = e;
    ldpc_code_desc desc = {N, M, row_ptr, col_idx, Z, MB, NB, shift};
    ldpc_code *code = NULL;
    LDPC(ldpc_code_create(&desc, 0, &code));
    int32_t nv, nc, dcmax, dvmax;
    int64_t ne;
    LDPC(ldpc_code_query(code, &nv, &nc, &ne, &dcmax, &dvmax));
    CHECK(nv == N && nc == M && ne == M * NB && dcmax == NB && dvmax == MB, "ldpc_code_query");

    /* all-zero codeword, int16 Q3 LLRs: +8 = LLR 1.0 */
    int16_t llr[F][N];
    for (int f = 0; f < F; ++f)
        for (int n = 0; n < N; ++n) llr[f][n] = (int16_t)(24 + (n * 7 + f * 3) % 17);
    llr[1][5] = -6;                                     /* one unreliable error */
    llr[2][17] = -4;                                    /* two errors in different rows */
    llr[2][70] = -3;
    for (int n = 0; n < N; n += 2) llr[3][n] = 2;       /* weak but correct */

    ldpc_decode_params p;
    memset(&p, 0, sizeof(p));
    p.max_iter = 20;
    p.early_stop = 1;
    p.variant = LDPC_MINSUM_OFFSET;
    p.offset_raw = 1;
    p.clamp_raw = 511;
    p.llr_type = LDPC_LLR_I16;
    p.msg_format = LDPC_MSG_COMPACT;
    p.schedule = LDPC_SCHED_SINGLESCAN;

    const int wpf = (N + 31) / 32;
    /* device entry point */
    size_t ws_bytes = 0;
    LDPC(ldpc_decode_workspace_size(code, F, &p, &ws_bytes));
    void *d_llr, *d_ws, *d_post;
    uint32_t *d_hb;
    uint8_t *d_ok;
    int32_t *d_it;
    CUDA(cudaMalloc(&d_llr, sizeof(llr)));
    CUDA(cudaMalloc(&d_ws, ws_bytes > 0 ? ws_bytes : 256));
    CUDA(cudaMalloc((void **)&d_hb, F * wpf * 4));
    CUDA(cudaMalloc(&d_post, F * N * 2));
    CUDA(cudaMalloc((void **)&d_ok, F));
    CUDA(cudaMalloc((void **)&d_it, F * 4));
    CUDA(cudaMemcpy(d_llr, llr, sizeof(llr), cudaMemcpyHostToDevice));
    LDPC(ldpc_decode_batch(code, &p, F, d_llr, d_hb, d_post, d_ok, d_it, d_ws, ws_bytes, NULL));
    CUDA(cudaDeviceSynchronize());
    uint32_t hb[F][(N + 31) / 32];
    int16_t post[F][N];
    uint8_t ok[F];
    int32_t it[F];
    CUDA(cudaMemcpy(hb, d_hb, sizeof(hb), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(post, d_post, sizeof(post), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(ok, d_ok, sizeof(ok), cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(it, d_it, sizeof(it), cudaMemcpyDeviceToHost));
    printf("device API: %d launch(es); iterations %d %d %d %d; syndrome_ok %d %d %d %d\n", ldpc_last_launch_count(),
           it[0], it[1], it[2], it[3], ok[0], ok[1], ok[2], ok[3]);
    for (int f = 0; f < F; ++f) {
        CHECK(ok[f] == 1, "frame %d not decoded", f);
        for (int w = 0; w < wpf; ++w) CHECK(hb[f][w] == 0u, "frame %d: hard bits word %d = %08x", f, w, hb[f][w]);
        for (int n = 0; n < N; ++n) CHECK(post[f][n] > 0, "frame %d: posterior %d = %d", f, n, post[f][n]);
    }
    CHECK(it[0] == 0 && it[3] == 0, "confident frames stop at iteration 0 (got %d, %d)", it[0], it[3]);
    CHECK(it[1] >= 1 && it[2] >= 1, "frames with errors need iterations (got %d, %d)", it[1], it[2]);

    /* host entry point: same outputs */
    size_t hws_bytes = 0;
    LDPC(ldpc_decode_host_workspace_size(code, F, &p, &hws_bytes));
    void *d_hws;
    CUDA(cudaMalloc(&d_hws, hws_bytes));
    uint32_t hb2[F][(N + 31) / 32];
    int16_t post2[F][N];
    uint8_t ok2[F];
    int32_t it2[F];
    cudaStream_t s;
    CUDA(cudaStreamCreate(&s));
    LDPC(ldpc_decode_batch_host(code, &p, F, llr, &hb2[0][0], &post2[0][0], ok2, it2, d_hws, hws_bytes, s));
    CUDA(cudaStreamSynchronize(s));
    CHECK(memcmp(hb, hb2, sizeof(hb)) == 0 && memcmp(post, post2, sizeof(post)) == 0 &&
              memcmp(ok, ok2, sizeof(ok)) == 0 && memcmp(it, it2, sizeof(it)) == 0,
          "host entry point differs from the device entry point");

    /* error counters (reading D14): all frames decoded to the transmitted codeword */
    int64_t *d_cnt, cnt[5];
    CUDA(cudaMalloc((void **)&d_cnt, sizeof(cnt)));
    CUDA(cudaMemset(d_cnt, 0, sizeof(cnt)));
    LDPC(ldpc_count_errors(code, F, d_hb, d_ok, d_it, d_cnt, NULL));
    CUDA(cudaMemcpy(cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost));
    CHECK(cnt[0] == 0 && cnt[1] == 0 && cnt[2] == 0 && cnt[3] == 0, "error counters %lld %lld %lld %lld",
          (long long)cnt[0], (long long)cnt[1], (long long)cnt[2], (long long)cnt[3]);
    CHECK(cnt[4] == (int64_t)(it[0] + it[1] + it[2] + it[3]), "iteration sum");

    /* error path: a NULL code is rejected with a reason */
    CHECK(ldpc_decode_workspace_size(NULL, F, &p, &ws_bytes) == LDPC_ERR_INVALID_ARG, "NULL code accepted");

    cudaStreamDestroy(s);
    cudaFree(d_cnt);
    cudaFree(d_hws);
    cudaFree(d_llr);
    cudaFree(d_ws);
    cudaFree(d_hb);
    cudaFree(d_post);
    cudaFree(d_ok);
    cudaFree(d_it);
    ldpc_code_destroy(code);
    printf("%s (libldpc version %d)\n", fails ? "FAILED" : "OK", ldpc_version());
    return fails ? 1 : 0;
}

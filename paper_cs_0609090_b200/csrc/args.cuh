// args.cuh -- kernel argument blocks shared by the host planner (ldpc_api.cu) and the
// kernel translation units (res_launch.cu, stream_launch.cu).  Plain data only.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "simd16.cuh"
#include "rowcore_types.cuh"

// Checked build (make checked -> build/checked/libldpc.so, LDPC_CHECKED defined): device-side
// bounds checks on every computed address of the hot loops (shared-memory gathers and REDs,
// TMEM row slots, posterior / state / output indices); a violation prints the condition and
// traps, so the launch fails with a CUDA error.  compute-sanitizer is closed on this GPU pool
// (profiles/r02_sanitizer_refusal.log); the GPU test suite run against this build is the
// memory-safety evidence (profiles/r02_checked_build_tests.log).  Compiled out otherwise.
#ifdef LDPC_CHECKED
#include <cstdio>
#define LDPC_CHECK(cond)                                                                          \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("LDPC_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define LDPC_CHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace ldpc {

constexpr int kMaxDC = 8;
constexpr int kQcMaxSB = 128;
constexpr int kQcGroups = 2;
constexpr int kQcMaxEnt = 1536;

// QC circulant table, passed by value (kernel parameter = constant bank).
struct QcTab {
    int nsb;                            // super-batches per iteration
    uint32_t Z4;                        // 4 * Z (bytes)
    int32_t e0[kQcMaxSB][kQcGroups];    // first entry of the base row handled by group g
    int32_t dc[kQcMaxSB][kQcGroups];    // its degree (0 = group idle in this super-batch)
    int32_t run_end[kQcMaxSB][kQcGroups];  // first later super-batch where the group's degree changes
    int16_t tcol[kQcMaxSB][kQcGroups];     // FMT_FULL: first TMEM column of slot b's messages in group g
    int16_t brow[kQcMaxSB][kQcGroups];     // base row of slot b in group g (message export)
    int nent;                           // entries in ent[]
    uint2 ent[kQcMaxEnt];               // (4 * shift, 4 * (j * Z)) per base-matrix entry
};

// barrier-free resident kernel, fixed buffer bases (ResArgs::fixed_bases): byte offset of buffer 1
constexpr uint32_t kAtomFixOff = 32768;

constexpr int kMaxSched = 64;   // per-iteration variant table of the resident kernels

struct ResArgs {
    int N, Np, M, npairs, nframes, K, Qsat, wpf;   // Np = N rounded up to 4; wpf = ceil(N/32)
    VarK vk;                       // check-node variant (constant over iterations)
    int nsched;                    // > 0: iteration k uses vk_sched[k-1] (lambda_k / beta_k)
    VarK vk_sched[kMaxSched];
    float alpha, beta;             // fp32 resident kernel: |L| = max(alpha*min - beta, 0)
    float alpha_sched[kMaxSched], beta_sched[kMaxSched];   // ... per iteration when nsched > 0
    const void *llr;
    uint32_t *hard_bits;
    int16_t *post;
    uint8_t *ok;
    int32_t *iters;
    uint32_t *ws;
    size_t slot_words;
    int nbatch;                       // CSR: colour batches (QC: unused, see QcTab::nsb)
    const int32_t *bptr;              // CSR: batch b = schedule positions [bptr[b], bptr[b+1])
    const uint32_t *colT;             // CSR: [kMaxDC][M] byte offsets 4*n of each edge
    const uint8_t *dcT;               // CSR: degree per schedule position
    const uint8_t *coldeg;            // [N] column degrees d_v(n) (barrier-free kernel's accumulator start)
    int Z;                            // QC circulant size
    int group_threads;                // QC: threads per group (128 with two groups)
    uint32_t tmem_cols;               // TMEM columns allocated per CTA
    int cols_per_group;               // TMEM columns used by one group of threads
    RegK rk;                          // register constants (simd16.cuh)
    uint32_t cpar;                    // row_parity constant (-(0x00010001), biased: -(0x40014001))
    int csr_smem, csr_dc;             // barrier-free kernel, general codes: colT rows [0, csr_dc) staged in smem
    int fixed_bases;                  // barrier-free kernel with early stop: second posterior buffer at the
                                      // fixed byte offset kAtomFixOff, shift / column table in shared memory
                                      // with buffer 0's address folded in (k_resident_atom.cuh)
    int dc_uniform;                   // general codes: the row degree if every row has it, else 0
    // message export (ldpc_decode_batch_messages): the exit messages L_mn rebuilt from each
    // row's state, int16 [nframes][E] in CSR edge order; nullptr = no export
    int16_t *msg_out;
    const int32_t *row_ptr;
    int64_t E;
};

struct StreamArgs {
    RegK rk;                     // register constants (simd16.cuh)
    int N, M, ntiles, nframes, K, Qsat, wpf;
    VarK vk;                     // check-node variant of this launch's iteration
    float alpha, beta;           // fp32 variant: |L| <= max(alpha*min - beta, 0)
    const int32_t *row_ptr, *col_idx;
    const uint4 *rowtab;         // [M][2]: up to 8 column indices per row; dc in bits 28-31 of word 0 (15 = wider row)
    const uint8_t *coldeg;       // [N] column degrees (integer path: accumulator start values)
    const void *llr;
    uint32_t *Z0;                // [tile][N][32]
    uint32_t *Lb[3];             // rotating posterior buffers [tile][N][32]
    uint32_t *st;                // [tile][words][M][32]
    uint32_t *synd;              // [tile][32]: syndrome-fail bits found during the current launch
    uint32_t *done;              // [tile][32]: frames frozen (early stop)
    int32_t *it_ws;              // [tile*TILE] iterations used per frame
    // fp32 on the pipelined kernel ("delta" accumulation, k_stream_pipe.cuh): the posterior
    // of iteration k lives in Lb[k & 1] and the compact state of iteration k in plane k & 1
    // (st, st2); 0 = the three rotating posterior buffers Lb[k % 3] and one state plane
    int f32delta;
    uint32_t *st2;
    int layered;                 // LDPC_SCHED_LAYERED on the streaming layout (k_stream_layered.cuh): one
                                 // posterior plane Lb[0], integer biased / fp32 plain floats
    uint8_t *ok_ws;              // [tile*TILE] syndrome ok per frame (frozen frames)
    uint32_t *hard_bits;
    void *post;
    uint8_t *ok;
    int32_t *iters;
    void *msg_out;               // message export: int16 / float [nframes][E], nullptr = none
    int64_t E;
};

// two-scan baseline (k_twoscan.cuh): column addressing and the per-edge message planes
struct TwoScanArgs {
    const int32_t *vptr;    // [N+1] column pointers
    const int32_t *vedge;   // [E] edge ids of column n, ascending row
    const int32_t *ecol;    // [E] column of edge e (CSR col_idx)
    uint32_t *msg;          // [tile][E][32] L_mn
    uint32_t *zv;           // [tile][E][32] Z_mn
    uint32_t *hb;           // [tile][N][2] (int pairs: lo, hi frames) or [tile][N] (fp32): hard-decision
                            // ballots of the posterior written by the variable pass (early stop)
    int64_t E;
    int max_dv;             // largest column degree (selects the variable-pass instantiation)
};

// persistent state formats (workspace words per row-pair)
// FMT_C16 : 3 words (A, B, W); magnitudes up to 2Q = 1022.
// FMT_1BIT: 2 words (X = bytes [A_lo, B_lo, A_hi, B_hi], W); magnitudes up to 2Q = 254.
// FMT_FULL: the §4 single-scan -- one word per EDGE, the previous message L_mn
//           itself (barrier-free resident kernel only; k_resident_atom.cuh).
enum { FMT_C16 = 0, FMT_1BIT = 1, FMT_FULL = 2 };

}  // namespace ldpc

/*
 * ldpc.h -- C ABI of the B200 single-scan min-sum LDPC decoder (libldpc.so).
 *
 * Implements the data-parallel hot path of X. Huang, "Single-Scan Min-Sum
 * Algorithms for Fast Decoding of LDPC Codes" (ITW 2006; /root/reference/PAPER.md,
 * cited as P:<line>):
 *   - the single-scan check-node update that forms Z_mn = Z_n - L_mn from the
 *     posterior and the previous check message (§4, Eq.(3)),
 *   - over the memory-efficient compact per-check state (A_m, B_m, ñ_m, s_mn) from
 *     which every L_mn is rebuilt (§5, Eq.(4)/(5)),
 *   - with the normalized / offset modifications,
 *   - hard decision and syndrome stop rule (§3),
 * decoding a batch of independent frames, using only check->variable addressing
 * (P:219-224).  Numeric readings of silent passages: DESIGN.md §3 (D1-D28).
 *
 * Conventions (all entry points):
 *   - Plain C types only.  `stream` is a cudaStream_t passed as void* (NULL =
 *     legacy default stream).
 *   - No exceptions cross the ABI; every call returns an ldpc_status.  On error
 *     nothing has been launched or written, and ldpc_last_error_detail() returns
 *     a thread-local human-readable reason.
 *   - The caller owns every buffer it passes.  The library owns only the
 *     ldpc_code object and the device copy of the code structure it holds.
 *   - ldpc_decode_batch() is asynchronous on `stream`: no host synchronisation,
 *     no allocation.  One code may be used concurrently from several streams /
 *     host threads provided each call has its own workspace and outputs.
 */
#ifndef LDPC_B200_LDPC_H
#define LDPC_B200_LDPC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ldpc_code ldpc_code;   /* opaque, immutable after create */

typedef enum {
    LDPC_OK = 0,
    LDPC_ERR_INVALID_ARG = 1,    /* NULL pointer, bad size, bad enum value, workspace too small */
    LDPC_ERR_INVALID_CODE = 2,   /* H violates the ldpc_code_desc rules below */
    LDPC_ERR_UNSUPPORTED = 3,    /* valid request outside what the kernels implement (see params) */
    LDPC_ERR_CUDA = 4,           /* a CUDA runtime call or launch failed (detail has the CUDA error) */
    LDPC_ERR_NO_MEMORY = 5       /* host or device allocation failed in ldpc_code_create */
} ldpc_status;

/* Parity-check matrix H (M x N, binary) -- PAPER.md P:90-106 (§2): N(m) is row m.
 * Rules (violations -> LDPC_ERR_INVALID_CODE):
 *   n_vars >= 2, n_checks >= 1; row_ptr[0] = 0, row_ptr non-decreasing, E = row_ptr[M];
 *   every col_idx in [0, N); columns strictly increasing within a row (no duplicates);
 *   every row degree |N(m)| >= 2 (Eq.(1) needs N(m)\n non-empty);
 *   every column degree |M(n)| >= 1.
 * Optional quasi-cyclic description (qc_z > 0): base matrix qc_rows x qc_cols with
 * M = qc_rows*qc_z, N = qc_cols*qc_z; qc_shift[i*qc_cols + j] = -1 (empty) or
 * s in [0, qc_z), meaning a 1 at (i*qc_z + r, j*qc_z + (r + s) mod qc_z) for every
 * r.  The CSR must equal the expansion of the shift table (else INVALID_CODE).
 * All pointers are HOST pointers, read during the call only. */
typedef struct {
    int32_t n_vars;            /* N */
    int32_t n_checks;          /* M */
    const int32_t *row_ptr;    /* host, M+1 entries */
    const int32_t *col_idx;    /* host, E entries, 0-based */
    int32_t qc_z;              /* 0 = not quasi-cyclic; else circulant size Z */
    int32_t qc_rows, qc_cols;  /* base matrix shape (ignored when qc_z == 0) */
    const int16_t *qc_shift;   /* host, qc_rows*qc_cols entries (ignored when qc_z == 0) */
} ldpc_code_desc;

/* Validate H, build the device-side structures (check->variable addressing for the
 * single-scan kernels, a conflict-free row schedule, the QC circulant tables, and the
 * variable->check column lists used only by the TWOSCAN baseline) on `cuda_device`.
 * Synchronous.  *out is set only on LDPC_OK. */
ldpc_status ldpc_code_create(const ldpc_code_desc *desc, int cuda_device, ldpc_code **out);

/* Free a code (NULL is a no-op).  The caller must ensure no decode using it is in flight. */
void ldpc_code_destroy(ldpc_code *code);

/* Sizes of a code: N, M, E = sum |N(m)|, max row degree, max column degree.  Any output may be NULL. */
ldpc_status ldpc_code_query(const ldpc_code *code, int32_t *n_vars, int32_t *n_checks, int64_t *n_edges,
                            int32_t *max_dc, int32_t *max_dv);

/* Channel LLR element types.  Integer LLRs are raw fixed-point values (the
 * library does not need the fraction bits): I16 is e.g. Q3 (LLR*8), I8 e.g. Q2. */
enum { LDPC_LLR_I16 = 0, LDPC_LLR_I8 = 1, LDPC_LLR_F32 = 2 };
/* Check-node variant (P:178-188 two-scan; P:338-353 single-scan compact form). */
enum { LDPC_MINSUM_OFFSET = 0,       /* |L| <= max(|L| - beta, 0); offset 0 = plain min-sum */
       LDPC_MINSUM_NORMALIZED = 1 }; /* |L| <= alpha |L|, 0 < alpha <= 1 (integer LLRs: floor, dyadic alpha) */
/* Persistent message format.  Both keep, per check row, the two
 * magnitudes A_m <= B_m, the position ñ_m and one sign bit s_mn per edge:
 *   COMPACT: magnitudes stored with 9+ bits (clamp Q <= 511 for integer LLRs);
 *   ONEBIT : "1-bit messages": the only per-edge persistent datum is the
 *            sign bit; magnitudes are stored as bytes (integer LLRs, Q <= 127). */
enum { LDPC_MSG_COMPACT = 0, LDPC_MSG_1BIT = 1,
       LDPC_MSG_FULL = 2 };   /* FULL: the §4 single-scan storing every L_mn (one
                                 16-bit value per edge per frame, on chip).  Integer LLRs,
                                 SINGLESCAN schedule, codes on the resident path with
                                 2Q(max_dv+1) < 16384 and the messages within the Tensor Memory
                                 budget (else LDPC_ERR_UNSUPPORTED).  Same outputs as COMPACT
                                 (P:338). */
/* Decoding schedule.
 *   SINGLESCAN: the paper's method -- flooding single-scan min-sum over the compact
 *               state (Eq.(3)); the default.
 *   TWOSCAN   : the two-scan min-sum of §3 the paper compares against
 *               (P:29-30): per-edge messages L_mn and Z_mn in device memory, a
 *               horizontal (check) and a vertical (variable) scan per iteration, both
 *               addressings.  Same outputs as SINGLESCAN (bit-exact for
 *               integer LLRs); requires msg_format COMPACT, row degree <= 8 and
 *               column degree <= 16 (else LDPC_ERR_UNSUPPORTED).  A baseline, not a
 *               fast path: it always uses the streaming (HBM) layout.
 *   LAYERED   : the Eq.(3) block with ONE in-place posterior array (the paper stores
 *               "Z_n, which are of N items"): rows are processed in ascending
 *               m and row m replaces its old message in the current posterior,
 *               Z_n <- (Z_n - L^(k-1)_mn) + L^(k)_mn, so it sees the updates of the rows
 *               before it (layered / Gauss-Seidel schedule, reading D25).  Not
 *               equivalent to two-scan; usually converges in fewer iterations.  The row
 *               order of H defines the schedule (QC codes: base row by base row).
 *               Codes whose posteriors fit in shared memory (e.g. N <= ~27000) run on the
 *               resident kernel; longer codes (and tuning.path = LDPC_PATH_STREAM) on the
 *               streaming layered kernel: one warp per 64-frame (F32: 32-frame) tile walks
 *               the rows in order -- correct at any size but latency-bound (the schedule is
 *               a chain of M dependent row updates per frame).  Per-iteration
 *               schedules: max_iter <= 64.  Row degree <= 8, else LDPC_ERR_UNSUPPORTED.  Integer and F32
 *               LLRs (F32 layered is bit-exact with a sequential implementation). */
enum { LDPC_SCHED_SINGLESCAN = 0, LDPC_SCHED_TWOSCAN = 1, LDPC_SCHED_LAYERED = 2 };

/* Optional plan overrides (kernel cross-checks and tuning).  A NULL ldpc_decode_params.tuning
 * or a zero field selects the automatic choice.  The library reads no environment variables:
 * the plan depends only on the call's arguments. */
enum { LDPC_PATH_AUTO = 0,               /* resident kernel when the code fits on chip, else streaming */
       LDPC_PATH_STREAM = 1,             /* force the streaming (HBM) kernels */
       LDPC_PATH_RESIDENT_BATCHED = 2 }; /* integer flooding: the resident kernel with conflict-free row
                                            batches and a barrier per batch (instead of shared atomics) */
typedef struct {
    int32_t path;            /* LDPC_PATH_* */
    int32_t resident_waves;  /* resident grid cap in waves of co-resident CTAs (0 = 64); larger
                                batches loop over frame pairs */
    int32_t stream_chunk_tiles; /* streaming: frame tiles decoded together through all iterations
                                   (0 = all tiles at once) */
    int32_t stream_register_kernels; /* streaming: 1 = the register kernels instead of the cp.async
                                        row pipeline (cross-check), 0 = automatic */
    int32_t host_chunks;     /* ldpc_decode_batch_host: frame chunks (0 = automatic) */
    int32_t host_streams;    /* ldpc_decode_batch_host: internal streams, 1..4 (0 = automatic) */
    int32_t resident_threads; /* general (non-QC) codes on the barrier-free resident kernel: threads
                                 per CTA, a multiple of 32 in [32, 256] (0 = automatic) */
    int32_t resident_fixed_bases; /* early stop on the barrier-free resident kernel (QC codes, and
                                     general codes whose column table is staged in shared memory):
                                     -1 = posterior buffer bases in registers (cross-check),
                                     0 = automatic (fixed bases, immediate-offset addressing, when
                                     4*N <= 32768 and it costs no occupancy) */
} ldpc_tuning;

typedef struct {
    int32_t max_iter;      /* >= 1: the iteration cap of P:174-175 */
    int32_t early_stop;    /* 0: run max_iter iterations; 1: per frame, stop at the first k >= 0
                              whose hard decision satisfies H x̂ = 0 (the k = 0 check is on the
                              channel LLRs; reading D10).  Outputs are frozen at that k. */
    int32_t variant;       /* LDPC_MINSUM_OFFSET | LDPC_MINSUM_NORMALIZED */
    int32_t offset_raw;    /* integer LLRs: offset beta in LSBs, >= 0 */
    float   offset_f;      /* F32 LLRs: offset beta, >= 0 (OFFSET variant) */
    float   alpha;         /* NORMALIZED variant: lambda in (0, 1]; integer LLRs: dyadic, floor(lambda|L|) */
    int32_t clamp_raw;     /* integer LLRs: magnitude clamp Q applied after the offset (reading
                              D6); 0 = default (511 for I16, 127 for I8).  Channel LLRs are
                              saturated to [-Q, Q] on load.  Requires 2*Q*(max_dv + 2) <= 32767
                              (posteriors are exact in 16-bit lanes), Q <= 511 (COMPACT) or
                              Q <= 127 (ONEBIT), else LDPC_ERR_UNSUPPORTED.  Codes too long for
                              the resident kernel (streaming kernels, and TWOSCAN) additionally
                              need 2*Q*(max_dv + 1) < 16384 (biased 16-bit lanes, D26).
                              Ignored for F32. */
    int32_t llr_type;      /* LDPC_LLR_I16 | LDPC_LLR_I8 | LDPC_LLR_F32 */
    int32_t msg_format;    /* LDPC_MSG_COMPACT | LDPC_MSG_1BIT | LDPC_MSG_FULL (1BIT and FULL
                              require integer LLRs).  F32 LLRs: row degree <= 16 (LAYERED:
                              <= 8); integer: row degree <= 8. */
    int32_t schedule;      /* LDPC_SCHED_SINGLESCAN (0, default) | _TWOSCAN | _LAYERED */
    /* Optional per-iteration variants (P:179 lambda_k, P:186 beta_k): HOST arrays of
     * max_iter entries, read during the call only; NULL = the constants above.
     *   offset_per_iter   integer LLRs: beta_k in LSBs (>= 0)
     *   offset_f_per_iter F32 LLRs: beta_k (>= 0)
     *   alpha_per_iter    lambda_k in (0, 1] (any variant; overrides alpha)
     * Integer LLRs with lambda != 1 (constant or per iteration) use floor(lambda |L|)
     * (reading D27) and require a dyadic lambda = a/2^s with s <= 8 and
     * a * 2Q(max_dv+2) < 65536, else LDPC_ERR_UNSUPPORTED.  The resident kernels take
     * schedules of up to 64 iterations (longer ones run on the streaming kernels;
     * LAYERED: LDPC_ERR_UNSUPPORTED). */
    const int32_t *offset_per_iter;
    const float   *offset_f_per_iter;
    const float   *alpha_per_iter;
    const ldpc_tuning *tuning;   /* HOST, optional (NULL = automatic), read during the call only */
} ldpc_decode_params;

/* Device workspace bytes needed by ldpc_decode_batch for n_frames frames. */
ldpc_status ldpc_decode_workspace_size(const ldpc_code *code, int64_t n_frames,
                                       const ldpc_decode_params *params, size_t *bytes);

/* Decode n_frames independent frames (n_frames = 0 is a no-op returning LDPC_OK).
 *   llr          device, [n_frames][N], element type per params->llr_type (row-major, frame-major)
 *   hard_bits    device, [n_frames][ceil(N/32)] uint32; bit n%32 of word n/32 is x̂_n
 *                (x̂_n = 1 iff Z_n <= 0); unused high bits of the last word are 0
 *   posteriors   device or NULL, [n_frames][N]: int16 (integer LLRs, same raw units as the
 *                input) or float (F32); the posterior Z^(k)_n at exit
 *   syndrome_ok  device, [n_frames] uint8: 1 iff H x̂^T = 0 at exit
 *   iterations_used device or NULL, [n_frames] int32: iterations run for the frame (D10)
 *   workspace    device, >= ldpc_decode_workspace_size() bytes, 256-byte aligned
 * Fully asynchronous on `stream`; all outputs are valid once the stream reaches this point.
 * Every path is deterministic: integer posteriors are exact, and F32 posteriors sum their
 * messages exactly (int64 on the 2^-34 grid) and round once (DESIGN.md §3 D28), so outputs
 * are bit-reproducible run to run and independent of batch composition.  F32 channel LLRs
 * and message magnitudes saturate at +-2^20 (D28).
 * Kernel choice (automatic, see ldpc_tuning): integer codes whose posterior double buffer
 * fits in shared memory decode resident (one launch, a frame pair per CTA) when the compact
 * state of a CTA's rows fits in the SM's Tensor Memory; other codes, and F32 flooding /
 * two-scan decodes, use the streaming kernels (one launch per iteration). */
ldpc_status ldpc_decode_batch(const ldpc_code *code, const ldpc_decode_params *params, int64_t n_frames,
                              const void *llr, uint32_t *hard_bits, void *posteriors,
                              uint8_t *syndrome_ok, int32_t *iterations_used,
                              void *workspace, size_t workspace_bytes, void *stream);

/* Parity / debug export: ldpc_decode_batch plus the check messages at exit.
 *   messages  device, [n_frames][E]: int16 (integer LLRs, raw input units) or float (F32);
 *             entry (f, e) is L_mn of edge e = (m, n) in the CSR order of H (row_ptr[m] + j),
 *             the message of the last iteration: for SINGLESCAN rebuilt from the row's
 *             persistent state as the next iteration would (L_mn = s_mn f(A_m, B_m, n, ñ_m),
 *             so the export pins A_m, B_m, s_mn and ñ_m wherever A_m != B_m),
 *             for TWOSCAN the stored per-edge message of the last horizontal scan.
 * Defined for frames that ran all max_iter iterations (iterations_used == max_iter); the
 * entries of frames that stopped early are unspecified.  The same workspace as
 * ldpc_decode_batch.  LAYERED: the messages of the last iteration's row updates, on the
 * streaming layered kernel (long codes, or tuning.path = LDPC_PATH_STREAM).
 * LDPC_ERR_UNSUPPORTED on the resident layered and the batched resident kernels
 * (tuning.path = LDPC_PATH_RESIDENT_BATCHED, or codes with 2Q(max_dv+1) >= 16384 on the
 * resident path). */
ldpc_status ldpc_decode_batch_messages(const ldpc_code *code, const ldpc_decode_params *params, int64_t n_frames,
                                       const void *llr, uint32_t *hard_bits, void *posteriors,
                                       uint8_t *syndrome_ok, int32_t *iterations_used, void *messages,
                                       void *workspace, size_t workspace_bytes, void *stream);

/* Device workspace bytes for ldpc_decode_batch_host (includes device staging of inputs/outputs). */
ldpc_status ldpc_decode_host_workspace_size(const ldpc_code *code, int64_t n_frames,
                                            const ldpc_decode_params *params, size_t *bytes);

/* Same as ldpc_decode_batch but llr / hard_bits / posteriors / syndrome_ok /
 * iterations_used are HOST pointers (pinned memory recommended).  Enqueues the
 * host->device copy, the decode and the device->host copies on `stream`, split in
 * frame chunks so copies overlap decoding; returns without synchronising -- the
 * host outputs are valid after cudaStreamSynchronize(stream).  Outputs are staged in the
 * workspace and copied back by the copy engines (kernels writing straight into mapped
 * host memory were measured slower: DESIGN.md §7).  The chunks run on internal streams of
 * the code object: concurrent calls on one code are accepted (their enqueues are
 * serialised by a lock) and execute one after the other. */
ldpc_status ldpc_decode_batch_host(const ldpc_code *code, const ldpc_decode_params *params, int64_t n_frames,
                                   const void *llr_host, uint32_t *hard_bits_host, void *posteriors_host,
                                   uint8_t *syndrome_ok_host, int32_t *iterations_used_host,
                                   void *workspace, size_t workspace_bytes, void *stream);

/* Error counters for the all-zero transmitted codeword (reading D14), accumulated
 * (atomically added) into counters[5] (device int64):
 *   [0] bit errors (set hard bits), [1] frame errors (any bit set), [2] undetected
 *   errors (syndrome_ok = 1 but bits != 0), [3] not converged (syndrome_ok = 0),
 *   [4] sum of iterations_used (iterations_used may be NULL: adds 0).
 * Asynchronous on `stream`. */
ldpc_status ldpc_count_errors(const ldpc_code *code, int64_t n_frames, const uint32_t *hard_bits,
                              const uint8_t *syndrome_ok, const int32_t *iterations_used,
                              int64_t *counters, void *stream);

/* Number of kernel launches the last successful decode call on this host thread
 * enqueued (for instrumentation). */
int32_t ldpc_last_launch_count(void);

const char *ldpc_status_string(ldpc_status status);
/* Thread-local detail of the most recent error on this host thread ("" if none). */
const char *ldpc_last_error_detail(void);
/* Library version as MAJOR*10000 + MINOR*100 + PATCH. */
int32_t ldpc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LDPC_B200_LDPC_H */

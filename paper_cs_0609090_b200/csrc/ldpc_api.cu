// ldpc_api.cu -- C ABI of libldpc.so (declarations and contracts: include/ldpc.h).
//
// Host side: validation of H (SPEC-style invariants), the
// device code structure (check->variable addressing only), the
// conflict-free row schedule / QC circulant table used by the resident kernel,
// path selection and launches.  No torch types, no allocation in decode calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ldpc.h"
#include "launch.h"
#include "simd16.cuh"

using namespace ldpc;

namespace {

thread_local std::string g_detail;
thread_local int32_t g_launches = 0;

ldpc_status fail(ldpc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_detail = buf;
    return s;
}

#define CUDA_TRY(expr)                                                                            \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess) return fail(LDPC_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

struct ldpc_code {
    int device = 0;
    int sm_count = 0;
    size_t smem_optin = 0;
    size_t smem_per_sm = 0;
    int N = 0, M = 0;
    int64_t E = 0;
    int max_dc = 0, max_dv = 0;
    int dc_uniform = 0;              // the row degree when H is row-regular, else 0
    // device CSR (stream kernels)
    int32_t *d_row_ptr = nullptr, *d_col_idx = nullptr;
    uint32_t *d_rowtab = nullptr;   // [M][8] padded column table (streaming kernels)
    // variable->check addressing, used only by the two-scan baseline
    int32_t *d_vptr = nullptr, *d_vedge = nullptr;
    uint8_t *d_coldeg = nullptr;     // [N] column degrees (max 255)
    // resident schedule
    bool qc = false;
    int Z = 0, mb = 0, nb = 0;
    int nbatch = 0, res_threads = 0, group_threads = 0;
    bool res_ok = false;        // resident path possible (smem, degrees)
    size_t res_smem = 0;
    QcTab *qtab = nullptr;      // host copy, passed by value to the kernel (constant bank)
    int32_t *d_bptr = nullptr;
    uint32_t *d_colT = nullptr;
    uint8_t *d_dcT = nullptr;
    // layered schedule (reading D25): batches of CONSECUTIVE variable-disjoint rows
    int nbatch_lay = 0, res_threads_lay = 0;
    QcTab *qtab_lay = nullptr;
    int32_t *d_bptr_lay = nullptr;
    uint32_t *d_colT_lay = nullptr;
    uint8_t *d_dcT_lay = nullptr;
    // barrier-free flooding kernel (k_resident_atom.cuh): row slots per thread
    int nbatch_atom = 0, res_threads_atom = 0;
    QcTab *qtab_atom = nullptr;
    int full_cols_qc = 0;            // FMT_FULL: TMEM columns per group (QC: sum of the group's row degrees)
    std::mutex host_mu;              // serialises ldpc_decode_batch_host calls (shared aux streams/events)
    cudaStream_t aux[4] = {nullptr, nullptr, nullptr, nullptr};      // host-API pipeline streams
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
};

// ------------------------------------------------------------------ create
static ldpc_status validate_desc(const ldpc_code_desc *d, std::vector<int> &coldeg) {
    if (!d || !d->row_ptr || !d->col_idx) return fail(LDPC_ERR_INVALID_ARG, "NULL descriptor or CSR pointer");
    const int N = d->n_vars, M = d->n_checks;
    if (N < 2 || M < 1) return fail(LDPC_ERR_INVALID_CODE, "need n_vars >= 2 and n_checks >= 1 (got %d, %d)", N, M);
    if (d->row_ptr[0] != 0) return fail(LDPC_ERR_INVALID_CODE, "row_ptr[0] = %d, must be 0", d->row_ptr[0]);
    coldeg.assign(N, 0);
    for (int m = 0; m < M; ++m) {
        const int32_t a = d->row_ptr[m], b = d->row_ptr[m + 1];
        if (b < a) return fail(LDPC_ERR_INVALID_CODE, "row_ptr decreases at row %d", m);
        if (b - a < 2) return fail(LDPC_ERR_INVALID_CODE, "row %d: degree %d < 2", m, b - a);
        for (int32_t e = a; e < b; ++e) {
            const int32_t c = d->col_idx[e];
            if (c < 0 || c >= N) return fail(LDPC_ERR_INVALID_CODE, "row %d: column %d out of range [0,%d)", m, c, N);
            if (e > a && c <= d->col_idx[e - 1]) {
                if (c == d->col_idx[e - 1]) return fail(LDPC_ERR_INVALID_CODE, "row %d: duplicate column %d", m, c);
                return fail(LDPC_ERR_INVALID_CODE, "row %d: columns not strictly increasing at %d", m, c);
            }
            coldeg[c]++;
        }
    }
    for (int n = 0; n < N; ++n)
        if (coldeg[n] == 0) return fail(LDPC_ERR_INVALID_CODE, "column %d has degree 0", n);
    if (d->qc_z > 0) {
        const int Z = d->qc_z;
        if (!d->qc_shift) return fail(LDPC_ERR_INVALID_ARG, "qc_z > 0 but qc_shift is NULL");
        if ((int64_t)d->qc_rows * Z != M || (int64_t)d->qc_cols * Z != N)
            return fail(LDPC_ERR_INVALID_CODE, "QC shape %dx%d (Z=%d) inconsistent with M=%d N=%d", d->qc_rows,
                        d->qc_cols, Z, M, N);
        std::vector<int32_t> row;
        for (int i = 0; i < d->qc_rows; ++i) {
            for (int j = 0; j < d->qc_cols; ++j) {
                const int s = d->qc_shift[(size_t)i * d->qc_cols + j];
                if (s < -1 || s >= Z) return fail(LDPC_ERR_INVALID_CODE, "QC shift (%d,%d) = %d out of range", i, j, s);
            }
            for (int r = 0; r < Z; ++r) {
                row.clear();
                for (int j = 0; j < d->qc_cols; ++j) {
                    const int s = d->qc_shift[(size_t)i * d->qc_cols + j];
                    if (s >= 0) row.push_back(j * Z + (r + s) % Z);
                }
                std::sort(row.begin(), row.end());
                const int m = i * Z + r;
                const int32_t a = d->row_ptr[m], b = d->row_ptr[m + 1];
                if ((int)row.size() != b - a || !std::equal(row.begin(), row.end(), d->col_idx + a))
                    return fail(LDPC_ERR_INVALID_CODE, "row %d differs from the QC shift-table expansion", m);
            }
        }
    }
    return LDPC_OK;
}

template <typename T>
static ldpc_status upload(T **dst, const T *src, size_t n) {
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc((void **)dst, n * sizeof(T));
    if (e != cudaSuccess) return fail(LDPC_ERR_NO_MEMORY, "cudaMalloc(%zu): %s", n * sizeof(T), cudaGetErrorString(e));
    if (src) CUDA_TRY(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
    return LDPC_OK;
}

static void free_code(ldpc_code *c) {
    if (!c) return;
    cudaFree(c->d_row_ptr);
    cudaFree(c->d_col_idx);
    cudaFree(c->d_rowtab);
    cudaFree(c->d_vptr);
    cudaFree(c->d_coldeg);
    cudaFree(c->d_vedge);
    delete c->qtab;
    cudaFree(c->d_bptr);
    cudaFree(c->d_colT);
    cudaFree(c->d_dcT);
    delete c->qtab_lay;
    delete c->qtab_atom;
    cudaFree(c->d_bptr_lay);
    cudaFree(c->d_colT_lay);
    cudaFree(c->d_dcT_lay);
    for (auto &s : c->aux)
        if (s) cudaStreamDestroy(s);
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    delete c;
}

extern "C" ldpc_status ldpc_code_create(const ldpc_code_desc *desc, int cuda_device, ldpc_code **out) {
    g_detail.clear();
    if (!out) return fail(LDPC_ERR_INVALID_ARG, "out is NULL");
    std::vector<int> coldeg;
    ldpc_status st = validate_desc(desc, coldeg);
    if (st != LDPC_OK) return st;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
        return fail(LDPC_ERR_CUDA, "CUDA device %d not available (%d devices)", cuda_device, ndev);
    DeviceGuard guard(cuda_device);
    ldpc_code *c = new ldpc_code();
    c->device = cuda_device;
    c->N = desc->n_vars;
    c->M = desc->n_checks;
    c->E = desc->row_ptr[c->M];
    for (int m = 0; m < c->M; ++m) c->max_dc = std::max(c->max_dc, desc->row_ptr[m + 1] - desc->row_ptr[m]);
    c->dc_uniform = c->max_dc;
    for (int m = 0; m < c->M; ++m)
        if (desc->row_ptr[m + 1] - desc->row_ptr[m] != c->max_dc) c->dc_uniform = 0;
    for (int n = 0; n < c->N; ++n) c->max_dv = std::max(c->max_dv, coldeg[n]);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) {
        free_code(c);
        return fail(LDPC_ERR_CUDA, "cudaGetDeviceProperties failed");
    }
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    c->smem_per_sm = prop.sharedMemPerMultiprocessor;
    if ((st = upload(&c->d_row_ptr, desc->row_ptr, (size_t)c->M + 1)) != LDPC_OK ||
        (st = upload(&c->d_col_idx, desc->col_idx, (size_t)c->E)) != LDPC_OK) {
        free_code(c);
        return st;
    }
    const int N = c->N, M = c->M;
    {
        // column-major edge lists M(n) (ascending row) for the two-scan variable pass
        std::vector<int32_t> vptr((size_t)N + 1, 0), vedge((size_t)c->E), fill((size_t)N, 0);
        for (int64_t e = 0; e < c->E; ++e) vptr[(size_t)desc->col_idx[e] + 1]++;
        for (int n = 0; n < N; ++n) vptr[(size_t)n + 1] += vptr[n];
        for (int m = 0; m < M; ++m)
            for (int32_t e = desc->row_ptr[m]; e < desc->row_ptr[m + 1]; ++e) {
                const int n = desc->col_idx[e];
                vedge[(size_t)vptr[n] + fill[n]++] = e;
            }
        std::vector<uint8_t> cd((size_t)N);
        for (int n = 0; n < N; ++n) cd[(size_t)n] = (uint8_t)std::min(coldeg[(size_t)n], 255);
        if ((st = upload(&c->d_coldeg, cd.data(), cd.size())) != LDPC_OK ||
            (st = upload(&c->d_vptr, vptr.data(), vptr.size())) != LDPC_OK ||
            (st = upload(&c->d_vedge, vedge.data(), vedge.size())) != LDPC_OK) {
            free_code(c);
            return st;
        }
    }
    {
        std::vector<uint32_t> rt((size_t)M * 8, 0u);
        for (int m = 0; m < M; ++m) {
            const int32_t a = desc->row_ptr[m], b = desc->row_ptr[m + 1];
            const int dc = b - a;
            if (dc <= 8)
                for (int32_t e = a; e < b; ++e) rt[(size_t)m * 8 + (e - a)] = (uint32_t)desc->col_idx[e];
            rt[(size_t)m * 8] |= (uint32_t)(dc <= 8 ? dc : 15) << 28;
        }
        if (N >= (1 << 28)) { free_code(c); return fail(LDPC_ERR_UNSUPPORTED, "n_vars >= 2^28"); }
        if ((st = upload(&c->d_rowtab, rt.data(), rt.size())) != LDPC_OK) { free_code(c); return st; }
    }
    // ---------- resident schedule (only when a frame pair's double buffer fits in shared memory)
    if (c->max_dc <= kMaxDC && (size_t)2 * N * 4 + 16384 <= c->smem_optin) {
        int nqent = 0;
        for (int i = 0; desc->qc_z > 0 && i < desc->qc_rows * desc->qc_cols; ++i) nqent += desc->qc_shift[i] >= 0;
        if (desc->qc_z > 0 && desc->qc_z <= 256 && desc->qc_rows <= kQcMaxSB && nqent <= kQcMaxEnt) {
            c->qc = true;
            c->Z = desc->qc_z;
            c->mb = desc->qc_rows;
            c->nb = desc->qc_cols;
            c->qtab = new QcTab();
            QcTab &t = *c->qtab;
            t.Z4 = 4u * (uint32_t)c->Z;
            std::vector<int> rstart(c->mb + 1, 0);
            std::vector<std::vector<int>> cols(c->mb);
            int e = 0;
            for (int i = 0; i < c->mb; ++i) {
                rstart[i] = e;
                for (int j = 0; j < c->nb; ++j) {
                    const int s = desc->qc_shift[(size_t)i * c->nb + j];
                    if (s < 0) continue;
                    t.ent[e] = make_uint2(4u * (uint32_t)s, 4u * (uint32_t)(j * c->Z));
                    cols[i].push_back(j);
                    ++e;
                }
            }
            t.nent = e;
            // super-batches: pairs of base rows with disjoint column blocks (their Z rows
            // each touch distinct variables), processed by two 128-thread groups at once.
            const int groups = c->Z <= 128 ? 2 : 1;
            std::vector<std::pair<int, int>> sb;
            if (groups == 2) {
                auto disjoint = [&](int x, int y) {
                    for (int u : cols[x])
                        for (int v : cols[y])
                            if (u == v) return false;
                    return true;
                };
                std::vector<std::pair<int, int>> best;
                size_t best_pairs = 0;
                uint64_t rs = 0x9E3779B97F4A7C15ull;
                for (int trial = 0; trial < 64; ++trial) {
                    std::vector<int> order(c->mb);
                    for (int i = 0; i < c->mb; ++i) order[i] = i;
                    if (trial) {
                        for (int i = c->mb - 1; i > 0; --i) {
                            rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17;
                            std::swap(order[i], order[rs % (uint64_t)(i + 1)]);
                        }
                    }
                    std::vector<char> used(c->mb, 0);
                    std::vector<std::pair<int, int>> cur;
                    size_t npairs_found = 0;
                    for (int ii = 0; ii < c->mb; ++ii) {
                        const int x = order[ii];
                        if (used[x]) continue;
                        used[x] = 1;
                        int y = -1;
                        for (int jj = ii + 1; jj < c->mb; ++jj)
                            if (!used[order[jj]] && disjoint(x, order[jj])) { y = order[jj]; break; }
                        if (y >= 0) { used[y] = 1; ++npairs_found; }
                        cur.emplace_back(x, y);
                    }
                    if (trial == 0 || npairs_found > best_pairs) { best = cur; best_pairs = npairs_found; }
                }
                sb = best;
            } else {
                for (int i = 0; i < c->mb; ++i) sb.emplace_back(i, -1);
            }
            // order super-batches by the groups' degrees so equal-degree runs are long
            std::stable_sort(sb.begin(), sb.end(), [&](const std::pair<int, int> &x, const std::pair<int, int> &y) {
                auto deg = [&](int i) { return i >= 0 ? (int)cols[i].size() : 0; };
                if (deg(x.first) != deg(y.first)) return deg(x.first) > deg(y.first);
                return deg(x.second) > deg(y.second);
            });
            t.nsb = (int)sb.size();
            for (int b = 0; b < t.nsb; ++b) {
                const int rows[2] = {sb[b].first, sb[b].second};
                for (int g = 0; g < kQcGroups; ++g) {
                    const int i = g < groups ? rows[g] : -1;
                    t.e0[b][g] = i >= 0 ? rstart[i] : 0;
                    t.dc[b][g] = i >= 0 ? (int)cols[i].size() : 0;
                    t.brow[b][g] = (int16_t)(i >= 0 ? i : 0);
                }
            }
            for (int g = 0; g < kQcGroups; ++g)
                for (int b = t.nsb - 1; b >= 0; --b)
                    t.run_end[b][g] = (b + 1 < t.nsb && t.dc[b + 1][g] == t.dc[b][g]) ? t.run_end[b + 1][g] : b + 1;
            c->nbatch = t.nsb;
            c->group_threads = groups == 2 ? 128 : ((c->Z + 31) / 32) * 32;
            c->res_threads = groups * c->group_threads;
            // layered: base rows in their natural order; consecutive base rows i, i+1 with
            // disjoint column blocks share a super-batch (same result as i then i+1)
            {
                c->qtab_lay = new QcTab(t);
                QcTab &u = *c->qtab_lay;
                auto disjoint = [&](int x, int y) {
                    for (int a : cols[x])
                        for (int b : cols[y])
                            if (a == b) return false;
                    return true;
                };
                int nsb = 0;
                for (int i = 0; i < c->mb;) {
                    const int j = (groups == 2 && i + 1 < c->mb && disjoint(i, i + 1)) ? i + 1 : -1;
                    const int rows[2] = {i, j};
                    for (int g = 0; g < kQcGroups; ++g) {
                        const int r = rows[g];
                        u.e0[nsb][g] = r >= 0 ? rstart[r] : 0;
                        u.dc[nsb][g] = r >= 0 ? (int)cols[r].size() : 0;
                        u.brow[nsb][g] = (int16_t)(r >= 0 ? r : 0);
                    }
                    ++nsb;
                    i += j >= 0 ? 2 : 1;
                }
                u.nsb = nsb;
                for (int g = 0; g < kQcGroups; ++g)
                    for (int b = u.nsb - 1; b >= 0; --b)
                        u.run_end[b][g] = (b + 1 < u.nsb && u.dc[b + 1][g] == u.dc[b][g]) ? u.run_end[b + 1][g] : b + 1;
                c->nbatch_lay = nsb;
                c->res_threads_lay = c->res_threads;
            }
            // barrier-free flooding: each group owns a list of base rows (thread r = circulant
            // row r); longest-processing-time assignment balances the groups' edge counts,
            // each list sorted by degree so equal-degree rows form one dispatch run
            {
                c->qtab_atom = new QcTab(t);
                QcTab &u = *c->qtab_atom;
                std::vector<int> order(c->mb);
                for (int i = 0; i < c->mb; ++i) order[i] = i;
                std::stable_sort(order.begin(), order.end(),
                                 [&](int x, int y) { return cols[x].size() > cols[y].size(); });
                std::vector<std::vector<int>> lists(groups);
                std::vector<size_t> load(groups, 0);
                for (int i : order) {
                    int gbest = 0;
                    for (int gg = 1; gg < groups; ++gg)
                        if (load[gg] < load[gbest]) gbest = gg;
                    lists[gbest].push_back(i);
                    load[gbest] += cols[i].size();
                }
                int nsb = 0;
                for (auto &l : lists) nsb = std::max(nsb, (int)l.size());
                for (int b = 0; b < nsb; ++b)
                    for (int g = 0; g < kQcGroups; ++g) {
                        const int r = (g < groups && b < (int)lists[g].size()) ? lists[g][b] : -1;
                        u.e0[b][g] = r >= 0 ? rstart[r] : 0;
                        u.dc[b][g] = r >= 0 ? (int)cols[r].size() : 0;
                        u.brow[b][g] = (int16_t)(r >= 0 ? r : 0);
                    }
                u.nsb = nsb;
                for (int g = 0; g < kQcGroups; ++g)
                    for (int b = u.nsb - 1; b >= 0; --b)
                        u.run_end[b][g] = (b + 1 < u.nsb && u.dc[b + 1][g] == u.dc[b][g]) ? u.run_end[b + 1][g] : b + 1;
                for (int g = 0; g < kQcGroups; ++g) {          // FMT_FULL column offsets per slot
                    int col = 0;
                    for (int b = 0; b < u.nsb; ++b) {
                        u.tcol[b][g] = (int16_t)col;
                        col += u.dc[b][g];
                    }
                    c->full_cols_qc = std::max(c->full_cols_qc, col);
                }
                c->nbatch_atom = nsb;
                c->res_threads_atom = c->res_threads;
            }
        } else {
            // greedy colouring: rows of one colour share no variable
            std::vector<std::vector<int>> classes;
            std::vector<std::vector<uint64_t>> used;   // per colour: bitset over variables
            std::vector<int> color(M);
            const size_t words = ((size_t)N + 63) / 64;
            for (int m = 0; m < M; ++m) {
                int cc = 0;
                for (;; ++cc) {
                    if (cc == (int)classes.size()) {
                        classes.emplace_back();
                        used.emplace_back(words, 0ull);
                    }
                    bool okc = true;
                    for (int32_t e = desc->row_ptr[m]; e < desc->row_ptr[m + 1] && okc; ++e) {
                        const int n = desc->col_idx[e];
                        if (used[cc][n >> 6] >> (n & 63) & 1ull) okc = false;
                    }
                    if (okc && classes[cc].size() < 256) break;
                }
                classes[cc].push_back(m);
                for (int32_t e = desc->row_ptr[m]; e < desc->row_ptr[m + 1]; ++e) {
                    const int n = desc->col_idx[e];
                    used[cc][n >> 6] |= 1ull << (n & 63);
                }
            }
            std::vector<int32_t> bptr(1, 0);
            std::vector<uint32_t> colT((size_t)kMaxDC * M, 0u);
            std::vector<uint8_t> dcT(M);
            int p = 0, maxb = 0;
            for (auto &cl : classes) {
                for (int m : cl) {
                    const int32_t a = desc->row_ptr[m], b = desc->row_ptr[m + 1];
                    dcT[p] = (uint8_t)(b - a);
                    for (int32_t e = a; e < b; ++e) colT[(size_t)(e - a) * M + p] = 4u * (uint32_t)desc->col_idx[e];
                    ++p;
                }
                bptr.push_back(p);
                maxb = std::max(maxb, (int)cl.size());
            }
            c->nbatch = (int)classes.size();
            c->res_threads = ((maxb + 31) / 32) * 32;
            if ((st = upload(&c->d_bptr, bptr.data(), bptr.size())) != LDPC_OK ||
                (st = upload(&c->d_colT, colT.data(), colT.size())) != LDPC_OK ||
                (st = upload(&c->d_dcT, dcT.data(), dcT.size())) != LDPC_OK) {
                free_code(c);
                return st;
            }
            // layered: maximal runs of consecutive, pairwise variable-disjoint rows in
            // ascending m (<= 256 rows), so a batch in parallel == its rows in order
            {
                std::vector<int32_t> lptr(1, 0);
                std::vector<uint32_t> lcol((size_t)kMaxDC * M, 0u);
                std::vector<uint8_t> ldc(M);
                std::vector<int> stamp(N, -1);
                int maxl = 0, cur = 0;
                for (int m = 0; m < M; ++m) {
                    bool clash = cur >= 256;
                    for (int32_t e = desc->row_ptr[m]; e < desc->row_ptr[m + 1] && !clash; ++e)
                        if (stamp[desc->col_idx[e]] == (int)lptr.size() - 1) clash = true;
                    if (clash) {
                        lptr.push_back(m);
                        cur = 0;
                    }
                    for (int32_t e = desc->row_ptr[m]; e < desc->row_ptr[m + 1]; ++e) {
                        stamp[desc->col_idx[e]] = (int)lptr.size() - 1;
                        lcol[(size_t)(e - desc->row_ptr[m]) * M + m] = 4u * (uint32_t)desc->col_idx[e];
                    }
                    ldc[m] = (uint8_t)(desc->row_ptr[m + 1] - desc->row_ptr[m]);
                    maxl = std::max(maxl, ++cur);
                }
                lptr.push_back(M);
                c->nbatch_lay = (int)lptr.size() - 1;
                c->res_threads_lay = ((maxl + 31) / 32) * 32;
                // barrier-free flooding: thread t owns rows t, t + T, ... (natural order tables)
                c->res_threads_atom = std::min(256, ((M + 31) / 32) * 32);
                c->nbatch_atom = (M + c->res_threads_atom - 1) / c->res_threads_atom;
                if ((st = upload(&c->d_bptr_lay, lptr.data(), lptr.size())) != LDPC_OK ||
                    (st = upload(&c->d_colT_lay, lcol.data(), lcol.size())) != LDPC_OK ||
                    (st = upload(&c->d_dcT_lay, ldc.data(), ldc.size())) != LDPC_OK) {
                    free_code(c);
                    return st;
                }
            }
        }
        c->res_smem = (size_t)2 * (((size_t)N + 3) & ~(size_t)3) * 4;
        c->res_ok = c->res_smem <= c->smem_optin && c->res_threads <= 256;
    }
    for (auto &s : c->aux)
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
            free_code(c);
            return fail(LDPC_ERR_CUDA, "cudaStreamCreate failed");
        }
    for (auto &e : c->ev)
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            free_code(c);
            return fail(LDPC_ERR_CUDA, "cudaEventCreate failed");
        }
    *out = c;
    return LDPC_OK;
}

extern "C" void ldpc_code_destroy(ldpc_code *code) {
    if (!code) return;
    DeviceGuard guard(code->device);
    free_code(code);
}

extern "C" ldpc_status ldpc_code_query(const ldpc_code *c, int32_t *n_vars, int32_t *n_checks, int64_t *n_edges,
                                       int32_t *max_dc, int32_t *max_dv) {
    if (!c) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    if (n_vars) *n_vars = c->N;
    if (n_checks) *n_checks = c->M;
    if (n_edges) *n_edges = c->E;
    if (max_dc) *max_dc = c->max_dc;
    if (max_dv) *max_dv = c->max_dv;
    return LDPC_OK;
}

// ------------------------------------------------------------------ planning
namespace {

enum Path { PATH_RESIDENT = 0, PATH_STREAM_I = 1, PATH_STREAM_F = 2 };

struct Plan {
    Path path;
    VarK vk{};                   // integer check-node variant (constant)
    std::vector<VarK> vks;       // per-iteration integer variants (empty: constant)
    std::vector<float> alphas, betafs;   // per-iteration fp32 lambda_k / beta_k (empty: constant)
    int sched = LDPC_SCHED_SINGLESCAN;
    int Q = 0, beta = 0, fmt = FMT_C16;
    float alpha = 1.f, betaf = 0.f;
    // resident
    bool lay = false;            // layered schedule (LDPC_SCHED_LAYERED)
    int kind = RES_BATCHED;      // resident kernel variant (launch.h)
    int threads = 0, nbatch = 0;
    size_t smem = 0;
    int grid = 0;
    size_t slot_words = 0;
    uint32_t tmem_cols = 0, tmem_cols_needed = 0;
    int cols_per_group = 0;
    int csr_smem = 0;            // barrier-free kernel, general codes: column table in shared memory
    int fixed_bases = 0;         // barrier-free kernel with early stop: fixed buffer bases
    // stream
    int tile = 64, ntiles = 0;
    size_t off_z0 = 0, off_lb[3] = {0, 0, 0}, off_st = 0, off_synd = 0, off_done = 0, off_it = 0, off_ok = 0;
    size_t off_msg = 0, off_zv = 0, off_hb = 0;   // two-scan: per-edge L_mn and Z_mn planes, hard-bit ballots
    size_t ws_bytes = 0;
    bool f32delta = false;       // fp32 delta accumulation (second state plane at off_st2)
    size_t off_st2 = 0;
    ldpc_tuning tn{};            // the call's plan overrides (zero = automatic)
};

// integer variant of one iteration: offset beta (LSBs), normalization lambda = na / 2^ns
// (dyadic, reading D27), clamp Q.  Returns false if lambda is not dyadic with ns <= 8.
bool make_vark(double lambda, int beta, int Q, VarK &v) {
    v = VarK{};
    if (lambda == 1.0) {
        v.norm = 0;
        v.nbeta2p1 = pack2(1 - 2 * beta, 1 - 2 * beta);
        v.q2p1 = pack2(2 * Q + 1, 2 * Q + 1);
        v.nb8 = pack2(0x8000 - 2 * beta, 0x8000 - 2 * beta);
        v.q2 = pack2(2 * Q, 2 * Q);
        return true;
    }
    for (int ns = 0; ns <= 8; ++ns) {
        const double x = lambda * (double)(1 << ns);
        if (x == (double)(int64_t)x) {
            v.norm = 1;
            v.na = (uint32_t)(int64_t)x;
            v.ns = (uint32_t)ns;
            const uint32_t lm = (0xFFFFu >> ns) & 0xFFFEu;
            v.nmask = lm | (lm << 16);
            v.nb2 = pack2(-2 * beta, -2 * beta);
            v.q2 = pack2(2 * Q, 2 * Q);
            return true;
        }
    }
    return false;
}

cudaError_t res_occupancy_any(const ldpc_code *c, const ldpc_decode_params *p, const struct Plan &pl, int *blocks) {
    return res_occupancy(c->qc, p->early_stop != 0, pl.fmt, p->llr_type == LDPC_LLR_I8, pl.kind, pl.smem,
                         c->smem_per_sm, pl.threads, blocks);
}

ldpc_status make_plan(const ldpc_code *c, int64_t F, const ldpc_decode_params *p, Plan &pl) {
    if (!c) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    if (!p) return fail(LDPC_ERR_INVALID_ARG, "params is NULL");
    if (F < 0) return fail(LDPC_ERR_INVALID_ARG, "n_frames < 0");
    if (F > INT32_MAX) return fail(LDPC_ERR_UNSUPPORTED, "n_frames > 2^31 - 1");
    if (p->max_iter < 1) return fail(LDPC_ERR_INVALID_ARG, "max_iter must be >= 1");
    if (p->early_stop != 0 && p->early_stop != 1) return fail(LDPC_ERR_INVALID_ARG, "early_stop must be 0 or 1");
    if (p->schedule != LDPC_SCHED_SINGLESCAN && p->schedule != LDPC_SCHED_TWOSCAN &&
        p->schedule != LDPC_SCHED_LAYERED)
        return fail(LDPC_ERR_INVALID_ARG, "bad schedule %d", p->schedule);
    pl.sched = p->schedule;
    if (p->tuning) pl.tn = *p->tuning;
    if (pl.tn.path < LDPC_PATH_AUTO || pl.tn.path > LDPC_PATH_RESIDENT_BATCHED)
        return fail(LDPC_ERR_INVALID_ARG, "bad tuning.path %d", pl.tn.path);
    if (pl.tn.resident_waves < 0 || pl.tn.stream_chunk_tiles < 0 || pl.tn.host_chunks < 0 || pl.tn.host_streams < 0 ||
        pl.tn.host_streams > 4 || pl.tn.resident_threads < 0 || pl.tn.resident_threads > 256 ||
        pl.tn.resident_threads % 32 != 0 || pl.tn.resident_fixed_bases < -1 || pl.tn.resident_fixed_bases > 0)
        return fail(LDPC_ERR_INVALID_ARG, "bad tuning value");
    if (pl.sched == LDPC_SCHED_TWOSCAN) {
        if (p->msg_format != LDPC_MSG_COMPACT)
            return fail(LDPC_ERR_UNSUPPORTED, "two-scan stores full per-edge messages: msg_format must be COMPACT");
        if (c->max_dc > 8) return fail(LDPC_ERR_UNSUPPORTED, "two-scan supports row degree <= 8 (max %d)", c->max_dc);
        if (c->max_dv > 16) return fail(LDPC_ERR_UNSUPPORTED, "two-scan supports column degree <= 16 (max %d)", c->max_dv);
    }
    if (p->msg_format != LDPC_MSG_COMPACT && p->msg_format != LDPC_MSG_1BIT && p->msg_format != LDPC_MSG_FULL)
        return fail(LDPC_ERR_INVALID_ARG, "bad msg_format %d", p->msg_format);
    if (p->variant != LDPC_MINSUM_OFFSET && p->variant != LDPC_MINSUM_NORMALIZED)
        return fail(LDPC_ERR_INVALID_ARG, "bad variant %d", p->variant);
    const float alpha0 = p->variant == LDPC_MINSUM_NORMALIZED ? p->alpha : 1.f;
    for (int k = 0; p->alpha_per_iter && k < p->max_iter; ++k)
        if (!(p->alpha_per_iter[k] > 0.f && p->alpha_per_iter[k] <= 1.f))
            return fail(LDPC_ERR_INVALID_ARG, "alpha_per_iter[%d] must be in (0,1]", k);
    if (p->variant == LDPC_MINSUM_NORMALIZED && !(p->alpha > 0.f && p->alpha <= 1.f))
        return fail(LDPC_ERR_INVALID_ARG, "alpha must be in (0,1]");
    if (p->llr_type == LDPC_LLR_F32) {
        if (p->msg_format != LDPC_MSG_COMPACT)
            return fail(LDPC_ERR_UNSUPPORTED, "1-bit and full per-edge message formats need integer LLRs");
        if (c->max_dc > 16) return fail(LDPC_ERR_UNSUPPORTED, "F32 path supports row degree <= 16 (max %d)", c->max_dc);
        if (p->variant == LDPC_MINSUM_OFFSET && !(p->offset_f >= 0.f))
            return fail(LDPC_ERR_INVALID_ARG, "offset_f must be >= 0");
        pl.alpha = alpha0;
        pl.betaf = p->variant == LDPC_MINSUM_OFFSET ? p->offset_f : 0.f;
        if (p->alpha_per_iter || p->offset_f_per_iter) {
            for (int k = 0; k < p->max_iter; ++k) {
                const float b = p->offset_f_per_iter ? p->offset_f_per_iter[k] : pl.betaf;
                if (!(b >= 0.f)) return fail(LDPC_ERR_INVALID_ARG, "offset_f_per_iter[%d] must be >= 0", k);
                pl.alphas.push_back(p->alpha_per_iter ? p->alpha_per_iter[k] : pl.alpha);
                pl.betafs.push_back(b);
            }
        }
        // fp32 flooding and two-scan decode on the streaming kernels, whose exact int64
        // accumulation (reading D28) is order-free; the layered schedule is resident
        pl.path = PATH_STREAM_F;
        if (pl.sched == LDPC_SCHED_LAYERED) {
            // layered schedule (D25): resident (k_resident_f32_lay, one posterior array) when the
            // code fits, else (or with tuning.path = STREAM) the streaming layered kernel
            if (c->max_dc > kMaxDC)
                return fail(LDPC_ERR_UNSUPPORTED, "layered schedule supports row degree <= %d", kMaxDC);
            pl.lay = true;
            if (c->res_ok && c->res_threads_lay <= 256 && pl.tn.path != LDPC_PATH_STREAM) {
                if (!pl.alphas.empty() && p->max_iter > kMaxSched)
                    return fail(LDPC_ERR_UNSUPPORTED, "per-iteration schedules support max_iter <= %d", kMaxSched);
                pl.path = PATH_RESIDENT;
                pl.kind = RES_F32_LAY;
            } else if (!pl.alphas.empty() && p->max_iter > kMaxSched) {
                return fail(LDPC_ERR_UNSUPPORTED, "layered per-iteration schedules support max_iter <= %d", kMaxSched);
            }
        }
        pl.tile = 32;
    } else if (p->llr_type == LDPC_LLR_I16 || p->llr_type == LDPC_LLR_I8) {
        if (p->offset_raw < 0 || p->offset_raw > 16383) return fail(LDPC_ERR_INVALID_ARG, "offset_raw out of range");
        if (c->max_dc > kMaxDC) return fail(LDPC_ERR_UNSUPPORTED, "integer paths support row degree <= %d (max %d)", kMaxDC, c->max_dc);
        pl.fmt = p->msg_format == LDPC_MSG_1BIT ? FMT_1BIT : (p->msg_format == LDPC_MSG_FULL ? FMT_FULL : FMT_C16);
        pl.Q = p->clamp_raw > 0 ? p->clamp_raw : (p->llr_type == LDPC_LLR_I16 ? 511 : 127);
        const int qmax = pl.fmt == FMT_1BIT ? 127 : 511;
        if (pl.Q > qmax) return fail(LDPC_ERR_UNSUPPORTED, "clamp Q=%d exceeds %d for this message format", pl.Q, qmax);
        if ((int64_t)2 * pl.Q * (c->max_dv + 2) > 32767)
            return fail(LDPC_ERR_UNSUPPORTED, "2*Q*(max_dv+2) = %lld > 32767: posteriors would overflow 16-bit lanes",
                        (long long)2 * pl.Q * (c->max_dv + 2));
        pl.beta = p->offset_raw;
        // integer variants (constant and per iteration); normalized needs a
        // dyadic lambda = na / 2^ns (reading D27) and 2|q| na < 2^16 per lane
        const int64_t qmax2 = (int64_t)2 * pl.Q * (c->max_dv + 2);
        auto vark = [&](double lam, int b, VarK &v) -> ldpc_status {
            if (b < 0 || b > 16383) return fail(LDPC_ERR_INVALID_ARG, "offset %d out of range", b);
            if (!make_vark(lam, b, pl.Q, v))
                return fail(LDPC_ERR_UNSUPPORTED, "integer normalized min-sum needs a dyadic lambda = a/2^s, s <= 8 "
                                                  "(got %.9g)", lam);
            if (v.norm && (int64_t)v.na * qmax2 >= 65536)
                return fail(LDPC_ERR_UNSUPPORTED, "lambda = %u/2^%u too fine for 16-bit lanes at Q=%d", v.na, v.ns, pl.Q);
            return LDPC_OK;
        };
        ldpc_status vs = vark(alpha0, pl.beta, pl.vk);
        if (vs != LDPC_OK) return vs;
        if (p->alpha_per_iter || p->offset_per_iter) {
            pl.vks.resize((size_t)p->max_iter);
            for (int k = 0; k < p->max_iter; ++k) {
                vs = vark(p->alpha_per_iter ? p->alpha_per_iter[k] : alpha0,
                          p->offset_per_iter ? p->offset_per_iter[k] : pl.beta, pl.vks[(size_t)k]);
                if (vs != LDPC_OK) return vs;
            }
        }
        // tuning.path = LDPC_PATH_STREAM routes integer decodes through the streaming kernels
        pl.path = (c->res_ok && pl.tn.path != LDPC_PATH_STREAM && pl.sched == LDPC_SCHED_SINGLESCAN) ? PATH_RESIDENT
                                                                                                   : PATH_STREAM_I;
        if (pl.sched == LDPC_SCHED_LAYERED) {
            // resident layered kernel when the code fits on chip, else (or with tuning.path =
            // STREAM) the streaming layered kernel (k_stream_layered.cuh: one warp per frame tile)
            pl.lay = true;
            if (c->res_ok && c->res_threads_lay <= 256 && pl.tn.path != LDPC_PATH_STREAM) {
                pl.path = PATH_RESIDENT;
            } else {
                pl.path = PATH_STREAM_I;
                if (!pl.vks.empty() && p->max_iter > kMaxSched)
                    return fail(LDPC_ERR_UNSUPPORTED, "layered per-iteration schedules support max_iter <= %d",
                                kMaxSched);
            }
        }
        // the streaming integer kernels (flooding, layered and two-scan) keep posteriors as
        // 2Z + 0x4000 per 16-bit lane (reading D26): needs 2Q(max_dv+1) < 0x4000
        if (pl.path == PATH_STREAM_I && (int64_t)2 * pl.Q * (c->max_dv + 1) >= 0x4000)
            return fail(LDPC_ERR_UNSUPPORTED, "streaming integer decode needs 2*Q*(max_dv+1) < 16384 (Q=%d, max_dv=%d)",
                        pl.Q, c->max_dv);
        pl.tile = 64;
    } else {
        return fail(LDPC_ERR_INVALID_ARG, "bad llr_type %d", p->llr_type);
    }
    const bool f32res = pl.kind == RES_F32_LAY;
    const int64_t npairs = f32res ? F : (F + 1) / 2;   // CTA work units: frame pairs (fp32: frames)
    if (pl.path == PATH_RESIDENT && !pl.vks.empty() && p->max_iter > kMaxSched) {
        if (pl.lay) return fail(LDPC_ERR_UNSUPPORTED, "per-iteration schedules support max_iter <= %d", kMaxSched);
        pl.path = PATH_STREAM_I;                         // the streaming kernels take any schedule length
        if ((int64_t)2 * pl.Q * (c->max_dv + 1) >= 0x4000)
            return fail(LDPC_ERR_UNSUPPORTED, "per-iteration schedules longer than %d iterations need the streaming "
                                              "kernels, which need 2*Q*(max_dv+1) < 16384", kMaxSched);
    }
    if (pl.path == PATH_RESIDENT) {
        // flooding uses the barrier-free atomic kernel when the biased 16-bit lanes cannot
        // overflow: 2 Q (max_dv + 1) < 0x4000 (k_resident_atom.cuh); tuning.path =
        // LDPC_PATH_RESIDENT_BATCHED selects the batched kernel
        const bool atom_ok = (int64_t)2 * pl.Q * (c->max_dv + 1) < 0x4000 && c->nbatch_atom > 0;
        if (!f32res)
            pl.kind = pl.lay ? RES_LAYERED
                             : ((atom_ok && pl.tn.path != LDPC_PATH_RESIDENT_BATCHED) ? RES_ATOM : RES_BATCHED);
        const bool atom_rows = pl.kind == RES_ATOM;   // barrier-free row ownership
        pl.threads = pl.lay ? c->res_threads_lay : (atom_rows ? c->res_threads_atom : c->res_threads);
        pl.nbatch = pl.lay ? c->nbatch_lay : (atom_rows ? c->nbatch_atom : c->nbatch);
        if (atom_rows && !c->qc && pl.tn.resident_threads > 0) {   // rows t, t + T, ... of a general code
            pl.threads = pl.tn.resident_threads;
            pl.nbatch = (c->M + pl.threads - 1) / pl.threads;
        }
        pl.smem = pl.lay ? c->res_smem / 2 : c->res_smem;   // layered: one posterior array
        // TMEM columns: 3 (COMPACT) or 2 (1BIT) per batch per 128-thread group; layered
        // general codes keep the state in shared memory instead ([3][M] words, by row)
        pl.cols_per_group = (pl.fmt == FMT_C16 ? 3 : 2) * pl.nbatch;
        if (pl.fmt == FMT_FULL) pl.cols_per_group = c->qc ? c->full_cols_qc : 8 * pl.nbatch;   // one word per edge
        bool lay_smem_over = false;
        if (pl.lay && !c->qc) {
            pl.cols_per_group = 0;
            pl.smem += (size_t)3 * c->M * 4;
            lay_smem_over = pl.smem > c->smem_optin;   // -> the streaming layered kernel below
        }
        const int groups = (pl.threads + 127) / 128;   // 128-thread TMEM lane slices
        uint32_t need = (uint32_t)(pl.cols_per_group * groups), cols = 32;
        while (cols < need) cols <<= 1;
        pl.tmem_cols_needed = cols;
        if (cols > 512 || lay_smem_over) {
            // more check rows per thread than an SM's 512 TMEM columns can hold state for:
            // the streaming kernels (state in HBM) take the decode where they apply
            if (pl.fmt == FMT_FULL)
                return fail(LDPC_ERR_UNSUPPORTED, "full per-edge messages need %u TMEM columns (> 512)", need);
            if (pl.lay && (!pl.vks.empty() || !pl.alphas.empty()) && p->max_iter > kMaxSched)
                return fail(LDPC_ERR_UNSUPPORTED, "layered per-iteration schedules support max_iter <= %d", kMaxSched);
            const bool f32 = p->llr_type == LDPC_LLR_F32;
            if (!f32 && (int64_t)2 * pl.Q * (c->max_dv + 1) >= 0x4000)
                return fail(LDPC_ERR_UNSUPPORTED, "compact state needs %u TMEM columns (> 512) and the streaming "
                                                  "kernels need 2*Q*(max_dv+1) < 16384", need);
            pl.path = f32 ? PATH_STREAM_F : PATH_STREAM_I;
            pl.kind = RES_BATCHED;
            pl.tile = f32 ? 32 : 64;
        }
    }
    // FULL per-edge messages exist only in the barrier-free resident kernel: checked after
    // every path switch above (long per-iteration schedules, TMEM fallback, forced streaming)
    if (pl.fmt == FMT_FULL && (pl.path != PATH_RESIDENT || pl.kind != RES_ATOM))
        return fail(LDPC_ERR_UNSUPPORTED, "full per-edge messages (LDPC_MSG_FULL) need the barrier-free resident "
                                          "kernel: SINGLESCAN schedule, a code on the resident path, at most %d "
                                          "iterations of per-iteration schedules and 2*Q*(max_dv+1) < 16384", kMaxSched);
    if (pl.path == PATH_RESIDENT) {
        const uint32_t cols = pl.tmem_cols_needed;
        pl.tmem_cols = cols;
        int blocks = 0;
        cudaError_t e = res_occupancy_any(c, p, pl, &blocks);
        if (e != cudaSuccess) return fail(LDPC_ERR_CUDA, "occupancy query: %s", cudaGetErrorString(e));
        blocks = std::min(blocks, (int)(512 / cols));     // TMEM capacity per SM
        // barrier-free kernel on a general (CSR) code: stage its [dc][M] column table in
        // shared memory (per-edge offsets become shared loads) when that costs no occupancy
        if (pl.kind == RES_ATOM && !c->qc && pl.fmt != FMT_FULL) {
            Plan ps = pl;
            ps.smem = pl.smem + (size_t)4 * c->max_dc * c->M;
            int bs = 0;
            if (ps.smem <= c->smem_optin && res_occupancy_any(c, p, ps, &bs) == cudaSuccess &&
                std::min(bs, (int)(512 / cols)) >= blocks) {
                pl.csr_smem = 1;
                pl.smem = ps.smem;
            }
        }
        // barrier-free kernel, early stop: buffer 1 at a fixed offset and the shift table (QC) or
        // column table (general codes, when it is staged in shared memory) after it with buffer
        // 0's address folded in, so the row scans address both buffers with immediate offsets
        // (k_resident_atom.cuh) -- when the buffer fits below the offset and it costs no occupancy
        if (pl.kind == RES_ATOM && (c->qc || pl.csr_smem) && p->early_stop && pl.fmt != FMT_FULL &&
            pl.tn.resident_fixed_bases == 0 && (size_t)4 * ((c->N + 3) & ~3) <= kAtomFixOff) {
            Plan ps = pl;
            const size_t np4 = (size_t)4 * ((c->N + 3) & ~3);
            const size_t tab = c->qc ? (size_t)8 * c->qtab_atom->nent : (size_t)4 * c->max_dc * c->M;
            ps.smem = kAtomFixOff + ((np4 + 7) & ~(size_t)7) + tab;
            int bs = 0;
            if (ps.smem <= c->smem_optin && res_occupancy_any(c, p, ps, &bs) == cudaSuccess &&
                std::min(bs, (int)(512 / cols)) >= blocks) {
                pl.fixed_bases = 1;
                pl.smem = ps.smem;
            }
        }
        if (blocks < 1) return fail(LDPC_ERR_UNSUPPORTED, "resident kernel does not fit on an SM");
        // One frame pair per CTA (grid = pairs, up to 64 waves): the block scheduler then
        // balances the SMs dynamically.  Measured against a persistent grid of `blocks x SMs`
        // CTAs looping over pairs: cfg2 2.91 -> 2.67 ms, cfg3 40.6 -> 35.9 ms.  The price is
        // one Z^(0) slot per CTA in the workspace; the 64-wave cap bounds it (cfg2: <= 0.9 GB)
        // for huge batches, whose CTAs then loop over pairs.  tuning.resident_waves sets the cap.
        const int waves = pl.tn.resident_waves > 0 ? pl.tn.resident_waves : 64;
        pl.grid = (int)std::min<int64_t>(std::max<int64_t>(npairs, 1), (int64_t)blocks * c->sm_count * waves);
        pl.slot_words = ((size_t)c->N + 63) & ~(size_t)63;
        pl.ws_bytes = align256((size_t)pl.grid * pl.slot_words * 4);
    } else {
        // streaming layout (also the fallback of a resident plan that does not fit in TMEM)
        pl.ntiles = (int)((F + pl.tile - 1) / pl.tile);
        const size_t plane = (size_t)pl.ntiles * c->N * 32 * 4;
        // fp32: the posterior planes hold int64 exact sums (reading D28)
        const size_t lplane = pl.path == PATH_STREAM_F ? 2 * plane : plane;
        const int sw = pl.path == PATH_STREAM_F ? 3 : (pl.fmt == FMT_C16 ? 3 : 2);
        size_t off = 0;
        pl.off_z0 = off; off += align256(plane);
        for (int i = 0; i < 3; ++i) { pl.off_lb[i] = off; off += align256(lplane); }
        if (pl.sched == LDPC_SCHED_TWOSCAN) {
            const size_t eplane = (size_t)pl.ntiles * (size_t)c->E * 32 * 4;
            pl.off_msg = off; off += align256(eplane);
            pl.off_zv = off; off += align256(eplane);
            pl.off_hb = off; off += align256((size_t)pl.ntiles * c->N * 8);
        } else {
            pl.off_st = off; off += align256((size_t)pl.ntiles * sw * c->M * 32 * 4);
        }
        // fp32 single-scan on the pipelined kernel (row degree <= 8): the delta accumulation
        // keeps a second compact-state plane (k_stream_pipe.cuh)
        pl.f32delta = pl.path == PATH_STREAM_F && pl.sched == LDPC_SCHED_SINGLESCAN && c->max_dc <= 8 &&
                      pl.tn.stream_register_kernels != 1;
        if (pl.f32delta) { pl.off_st2 = off; off += align256((size_t)pl.ntiles * sw * c->M * 32 * 4); }
        pl.off_synd = off; off += align256((size_t)pl.ntiles * 32 * 4);
        pl.off_done = off; off += align256((size_t)pl.ntiles * 32 * 4);
        pl.off_it = off; off += align256((size_t)pl.ntiles * pl.tile * 4);
        pl.off_ok = off; off += align256((size_t)pl.ntiles * pl.tile);
        pl.ws_bytes = off;
    }
    return LDPC_OK;
}

cudaError_t run_resident(const ldpc_code *c, const Plan &pl, const ldpc_decode_params *p, int64_t F,
                         const void *llr, uint32_t *hb, void *post, uint8_t *ok, int32_t *it, void *msg, void *ws,
                         cudaStream_t s) {
    ResArgs a{};
    a.msg_out = (int16_t *)msg;
    a.row_ptr = c->d_row_ptr;
    a.E = c->E;
    a.N = c->N;
    a.Np = (c->N + 3) & ~3;
    a.M = c->M;
    a.npairs = (int)((F + 1) / 2);
    a.nframes = (int)F;
    a.K = p->max_iter;
    a.Qsat = pl.Q;
    a.wpf = (c->N + 31) / 32;
    a.vk = pl.vk;
    a.nsched = (int)pl.vks.size();
    for (size_t k = 0; k < pl.vks.size(); ++k) a.vk_sched[k] = pl.vks[k];
    a.llr = llr;
    a.hard_bits = hb;
    a.post = (int16_t *)post;
    a.ok = ok;
    a.iters = it;
    a.ws = (uint32_t *)ws;
    a.slot_words = pl.slot_words;
    a.nbatch = pl.nbatch;
    const bool natural = pl.kind != RES_BATCHED;   // layered / atom: row tables in natural order
    a.bptr = pl.lay ? c->d_bptr_lay : c->d_bptr;
    a.colT = natural ? c->d_colT_lay : c->d_colT;
    a.dcT = natural ? c->d_dcT_lay : c->d_dcT;
    a.cpar = pl.kind == RES_ATOM ? 0xBFFFC000u : 0xFFFEFFFFu;   // -(bias + 1) per lane (atom: bias 0x3FFF)
    a.csr_smem = pl.csr_smem;
    a.fixed_bases = pl.fixed_bases;
    a.dc_uniform = c->dc_uniform;
    a.csr_dc = c->max_dc;
    a.alpha = pl.alpha;
    a.beta = pl.betaf;
    if (pl.kind == RES_F32_LAY && !pl.alphas.empty()) {
        a.nsched = (int)pl.alphas.size();
        for (size_t k = 0; k < pl.alphas.size(); ++k) {
            a.alpha_sched[k] = pl.alphas[k];
            a.beta_sched[k] = pl.betafs[k];
        }
    }
    a.coldeg = c->d_coldeg;
    a.Z = c->Z;
    a.group_threads = c->group_threads;
    a.tmem_cols = pl.tmem_cols;
    a.cols_per_group = pl.cols_per_group;
    a.rk = make_regk();
    static const QcTab empty_tab{};
    const QcTab *qt = (pl.kind == RES_LAYERED || pl.kind == RES_F32_LAY) ? c->qtab_lay
                                                                          : (pl.kind == RES_ATOM ? c->qtab_atom : c->qtab);
    cudaError_t e = res_launch(c->qc, p->early_stop != 0, pl.fmt, p->llr_type == LDPC_LLR_I8, pl.kind, pl.grid,
                               pl.threads, pl.smem, a, qt ? *qt : empty_tab, s);
    ++g_launches;
    return e;
}

cudaError_t run_stream(const ldpc_code *c, const Plan &pl, const ldpc_decode_params *p, int64_t F, const void *llr,
                       uint32_t *hb, void *post, uint8_t *ok, int32_t *it, void *msg, void *ws, cudaStream_t s) {
    char *w = (char *)ws;
    StreamArgs a{};
    a.msg_out = msg;
    a.E = c->E;
    a.N = c->N;
    a.M = c->M;
    a.ntiles = pl.ntiles;
    a.nframes = (int)F;
    a.K = p->max_iter;
    a.Qsat = pl.Q;
    a.wpf = (c->N + 31) / 32;
    a.vk = pl.vk;
    a.alpha = pl.alpha;
    a.rk = make_regk();
    a.beta = pl.betaf;
    a.row_ptr = c->d_row_ptr;
    a.col_idx = c->d_col_idx;
    a.rowtab = (const uint4 *)c->d_rowtab;
    a.coldeg = c->d_coldeg;
    a.llr = llr;
    a.Z0 = (uint32_t *)(w + pl.off_z0);
    for (int i = 0; i < 3; ++i) a.Lb[i] = (uint32_t *)(w + pl.off_lb[i]);
    a.st = (uint32_t *)(w + pl.off_st);
    a.f32delta = pl.f32delta ? 1 : 0;
    a.st2 = pl.f32delta ? (uint32_t *)(w + pl.off_st2) : nullptr;
    a.synd = (uint32_t *)(w + pl.off_synd);
    a.done = (uint32_t *)(w + pl.off_done);
    a.it_ws = (int32_t *)(w + pl.off_it);
    a.ok_ws = (uint8_t *)(w + pl.off_ok);
    a.hard_bits = hb;
    a.post = post;
    a.ok = ok;
    a.iters = it;
    StreamRun r{};
    r.pair = pl.path == PATH_STREAM_I;
    r.i8 = p->llr_type == LDPC_LLR_I8;
    r.fmt = pl.fmt;
    r.es = p->early_stop != 0;
    r.max_iter = p->max_iter;
    r.max_dc = c->max_dc;
    r.ntiles = pl.ntiles;
    r.flags_bytes = pl.off_it - pl.off_synd;
    r.vk_sched = pl.vks.empty() ? nullptr : pl.vks.data();
    r.alpha_sched = pl.alphas.empty() ? nullptr : pl.alphas.data();
    r.beta_sched = pl.betafs.empty() ? nullptr : pl.betafs.data();
    // L2 chunking (opt-in, tuning.stream_chunk_tiles = tiles per chunk): measured SLOWER on
    // cfg4/cfg5 at every chunk size (the streaming kernels are issue/latency-
    // bound, not HBM-bound, and chunks add launch tails), so all tiles run together by default.
    r.chunk_tiles = pl.tn.stream_chunk_tiles;
    r.register_kernels = pl.tn.stream_register_kernels == 1;
    r.layered = pl.lay;
    a.layered = pl.lay ? 1 : 0;
    int32_t n = 0;
    cudaError_t e;
    if (pl.sched == LDPC_SCHED_TWOSCAN) {
        TwoScanArgs t{};
        t.vptr = c->d_vptr;
        t.vedge = c->d_vedge;
        t.ecol = c->d_col_idx;
        t.msg = (uint32_t *)(w + pl.off_msg);
        t.zv = (uint32_t *)(w + pl.off_zv);
        t.hb = (uint32_t *)(w + pl.off_hb);
        t.E = c->E;
        t.max_dv = c->max_dv;
        e = twoscan_run(a, t, r, s, &n);
    } else {
        e = stream_run(a, r, s, &n);
    }
    g_launches += n;
    return e;
}

ldpc_status decode_device(const ldpc_code *c, const ldpc_decode_params *p, int64_t F, const void *llr, uint32_t *hb,
                          void *post, uint8_t *ok, int32_t *it, void *ws, size_t wsb, cudaStream_t s,
                          const Plan &pl, void *msg = nullptr) {
    if (F == 0) return LDPC_OK;
    if (msg && pl.path == PATH_RESIDENT && pl.kind != RES_ATOM)
        return fail(LDPC_ERR_UNSUPPORTED, "message export needs the SINGLESCAN flooding kernels (barrier-free resident "
                                          "or streaming) or TWOSCAN; not the batched / layered resident kernels");
    if (!llr || !hb || !ok) return fail(LDPC_ERR_INVALID_ARG, "llr, hard_bits and syndrome_ok must be non-NULL");
    if (!ws || wsb < pl.ws_bytes)
        return fail(LDPC_ERR_INVALID_ARG, "workspace too small: %zu < %zu bytes", wsb, pl.ws_bytes);
    if (((uintptr_t)ws & 255) != 0) return fail(LDPC_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
    cudaError_t e = pl.path == PATH_RESIDENT ? run_resident(c, pl, p, F, llr, hb, post, ok, it, msg, ws, s)
                                             : run_stream(c, pl, p, F, llr, hb, post, ok, it, msg, ws, s);
    if (e != cudaSuccess) return fail(LDPC_ERR_CUDA, "launch failed: %s", cudaGetErrorString(e));
    return LDPC_OK;
}

}  // namespace

extern "C" ldpc_status ldpc_decode_workspace_size(const ldpc_code *code, int64_t n_frames,
                                                  const ldpc_decode_params *params, size_t *bytes) {
    g_detail.clear();
    if (!bytes) return fail(LDPC_ERR_INVALID_ARG, "bytes is NULL");
    if (!code) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    DeviceGuard guard(code->device);
    Plan pl;
    ldpc_status st = make_plan(code, n_frames, params, pl);
    if (st != LDPC_OK) return st;
    *bytes = n_frames == 0 ? 0 : pl.ws_bytes;
    return LDPC_OK;
}

extern "C" ldpc_status ldpc_decode_batch(const ldpc_code *code, const ldpc_decode_params *params, int64_t n_frames,
                                         const void *llr, uint32_t *hard_bits, void *posteriors,
                                         uint8_t *syndrome_ok, int32_t *iterations_used, void *workspace,
                                         size_t workspace_bytes, void *stream) {
    g_detail.clear();
    g_launches = 0;
    if (!code) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    DeviceGuard guard(code->device);
    Plan pl;
    ldpc_status st = make_plan(code, n_frames, params, pl);
    if (st != LDPC_OK) return st;
    return decode_device(code, params, n_frames, llr, hard_bits, posteriors, syndrome_ok, iterations_used, workspace,
                         workspace_bytes, (cudaStream_t)stream, pl);
}

extern "C" ldpc_status ldpc_decode_batch_messages(const ldpc_code *code, const ldpc_decode_params *params,
                                                  int64_t n_frames, const void *llr, uint32_t *hard_bits,
                                                  void *posteriors, uint8_t *syndrome_ok, int32_t *iterations_used,
                                                  void *messages, void *workspace, size_t workspace_bytes,
                                                  void *stream) {
    g_detail.clear();
    g_launches = 0;
    if (!code) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    if (!messages && n_frames > 0) return fail(LDPC_ERR_INVALID_ARG, "messages is NULL");
    DeviceGuard guard(code->device);
    Plan pl;
    ldpc_status st = make_plan(code, n_frames, params, pl);
    if (st != LDPC_OK) return st;
    return decode_device(code, params, n_frames, llr, hard_bits, posteriors, syndrome_ok, iterations_used, workspace,
                         workspace_bytes, (cudaStream_t)stream, pl, messages);
}

// ------------------------------------------------------------------ host I/O
namespace {
struct HostLayout {
    int64_t chunk = 0, nchunks = 0;
    int nstreams = 1;
    size_t elt = 2, post_elt = 2, wpf = 0;
    size_t off_llr = 0, off_hb = 0, off_post = 0, off_ok = 0, off_it = 0, off_ws[4] = {0, 0, 0, 0};
    size_t chunk_ws = 0, total = 0;
    Plan pl;                         // the plan of a full chunk (reused by every full chunk)
};

// Host-buffer decode: H2D copy, decode and D2H copies of frame chunks round-robin on up to
// four streams, so the copies of one chunk overlap the decode of others.  Up to 16 chunks of
// >= 512 frames (resident) / >= 64 frames (streaming) on up to 4 streams measured best
// (tools/sweep_e2e.py); ldpc_tuning.host_chunks / host_streams override.
ldpc_status host_layout(const ldpc_code *c, int64_t F, const ldpc_decode_params *p, HostLayout &h) {
    Plan pf;
    ldpc_status st0 = make_plan(c, F, p, pf);
    if (st0 != LDPC_OK) return st0;
    // chunks of >= 512 frames (resident kernels) or >= one 64-frame tile (streaming), <= 16:
    // every chunk costs ~25 us of host enqueue (one H2D, the decode, four D2H copies), which
    // small batches cannot hide (cfg1, 1024 frames: 2 chunks 0.147 ms, 4 chunks 0.178 ms)
    const int64_t min_chunk = pf.path == PATH_RESIDENT ? 512 : 64;
    h.nchunks = std::max<int64_t>(1, std::min<int64_t>(16, F / min_chunk));
    if (pf.tn.host_chunks > 0) h.nchunks = pf.tn.host_chunks;
    h.chunk = (F + h.nchunks - 1) / h.nchunks;
    h.chunk = ((h.chunk + 63) / 64) * 64;
    if (h.chunk == 0) h.chunk = 64;
    h.nchunks = (F + h.chunk - 1) / h.chunk;
    Plan &pl = h.pl;
    ldpc_status st = make_plan(c, h.chunk, p, pl);
    if (st != LDPC_OK) return st;
    h.elt = p->llr_type == LDPC_LLR_F32 ? 4 : (p->llr_type == LDPC_LLR_I8 ? 1 : 2);
    h.post_elt = p->llr_type == LDPC_LLR_F32 ? 4 : 2;
    h.wpf = ((size_t)c->N + 31) / 32;
    size_t off = 0;
    h.off_llr = off; off += align256((size_t)F * c->N * h.elt);
    h.off_hb = off; off += align256((size_t)F * h.wpf * 4);
    h.off_post = off; off += align256((size_t)F * c->N * h.post_elt);
    h.off_ok = off; off += align256((size_t)F);
    h.off_it = off; off += align256((size_t)F * 4);
    h.nstreams = (int)std::min<int64_t>(h.nchunks, 4);
    if (pf.tn.host_streams > 0) h.nstreams = pf.tn.host_streams;
    h.chunk_ws = pl.ws_bytes;
    for (int i = 0; i < h.nstreams; ++i) { h.off_ws[i] = off; off += align256(pl.ws_bytes); }
    h.total = off;
    return LDPC_OK;
}
}  // namespace

extern "C" ldpc_status ldpc_decode_host_workspace_size(const ldpc_code *code, int64_t n_frames,
                                                       const ldpc_decode_params *params, size_t *bytes) {
    g_detail.clear();
    if (!bytes || !code) return fail(LDPC_ERR_INVALID_ARG, "NULL argument");
    DeviceGuard guard(code->device);
    if (n_frames == 0) { *bytes = 0; return LDPC_OK; }
    HostLayout h;
    ldpc_status st = host_layout(code, n_frames, params, h);
    if (st != LDPC_OK) return st;
    *bytes = h.total;
    return LDPC_OK;
}

extern "C" ldpc_status ldpc_decode_batch_host(const ldpc_code *code, const ldpc_decode_params *params,
                                              int64_t n_frames, const void *llr_host, uint32_t *hard_bits_host,
                                              void *posteriors_host, uint8_t *syndrome_ok_host,
                                              int32_t *iterations_used_host, void *workspace, size_t workspace_bytes,
                                              void *stream) {
    g_detail.clear();
    g_launches = 0;
    if (!code) return fail(LDPC_ERR_INVALID_ARG, "code is NULL");
    if (n_frames == 0) return LDPC_OK;
    if (!llr_host || !hard_bits_host || !syndrome_ok_host)
        return fail(LDPC_ERR_INVALID_ARG, "llr, hard_bits and syndrome_ok must be non-NULL");
    DeviceGuard guard(code->device);
    HostLayout h;
    ldpc_status st = host_layout(code, n_frames, params, h);
    if (st != LDPC_OK) return st;
    if (!workspace || workspace_bytes < h.total)
        return fail(LDPC_ERR_INVALID_ARG, "workspace too small: %zu < %zu bytes", workspace_bytes, h.total);
    if (((uintptr_t)workspace & 255) != 0) return fail(LDPC_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
    char *w = (char *)workspace;
    cudaStream_t us = (cudaStream_t)stream;
    // the internal streams and events belong to the code: one enqueue at a time (the work
    // itself stays asynchronous; concurrent callers' decodes are ordered on those streams)
    std::lock_guard<std::mutex> lock(const_cast<ldpc_code *>(code)->host_mu);
    CUDA_TRY(cudaEventRecord(code->ev[0], us));
    for (int i = 0; i < h.nstreams; ++i) CUDA_TRY(cudaStreamWaitEvent(code->aux[i], code->ev[0], 0));
    int32_t launches = 0;
    const int N = code->N;
    for (int64_t ci = 0; ci < h.nchunks; ++ci) {
        const int si = (int)(ci % h.nstreams);
        cudaStream_t s = code->aux[si];
        const int64_t f0 = ci * h.chunk, nf = std::min<int64_t>(h.chunk, n_frames - f0);
        char *dl = w + h.off_llr + (size_t)f0 * N * h.elt;
        uint32_t *dhb = (uint32_t *)(w + h.off_hb) + (size_t)f0 * h.wpf;
        char *dpost = posteriors_host ? w + h.off_post + (size_t)f0 * N * h.post_elt : nullptr;
        uint8_t *dok = (uint8_t *)(w + h.off_ok) + f0;
        int32_t *dit = iterations_used_host ? (int32_t *)(w + h.off_it) + f0 : nullptr;
        CUDA_TRY(cudaMemcpyAsync(dl, (const char *)llr_host + (size_t)f0 * N * h.elt, (size_t)nf * N * h.elt,
                                 cudaMemcpyHostToDevice, s));
        Plan tail;
        if (nf != h.chunk && (st = make_plan(code, nf, params, tail)) != LDPC_OK) return st;
        g_launches = 0;
        st = decode_device(code, params, nf, dl, dhb, dpost, dok, dit, w + h.off_ws[si], h.chunk_ws, s,
                           nf == h.chunk ? h.pl : tail);
        if (st != LDPC_OK) return st;
        launches += g_launches;
        CUDA_TRY(cudaMemcpyAsync(hard_bits_host + (size_t)f0 * h.wpf, dhb, (size_t)nf * h.wpf * 4,
                                 cudaMemcpyDeviceToHost, s));
        if (dpost)
            CUDA_TRY(cudaMemcpyAsync((char *)posteriors_host + (size_t)f0 * N * h.post_elt, dpost,
                                     (size_t)nf * N * h.post_elt, cudaMemcpyDeviceToHost, s));
    }
    for (int i = 0; i < h.nstreams; ++i) {
        CUDA_TRY(cudaEventRecord(code->ev[1 + i], code->aux[i]));
        CUDA_TRY(cudaStreamWaitEvent(us, code->ev[1 + i], 0));
    }
    // the per-frame flags and iteration counts (a few KB) leave in one copy each once every
    // chunk has decoded: per chunk, these small copies cost the bidirectional PCIe pipeline
    // a fixed overhead each (cfg2 e2e 3.57 -> 3.29 ms; moving the hard bits here too was
    // slower, 3.47 ms: their 7.7 MB then trail the last decode -- DESIGN.md §7)
    CUDA_TRY(cudaMemcpyAsync(syndrome_ok_host, w + h.off_ok, (size_t)n_frames, cudaMemcpyDeviceToHost, us));
    if (iterations_used_host)
        CUDA_TRY(cudaMemcpyAsync(iterations_used_host, w + h.off_it, (size_t)n_frames * 4, cudaMemcpyDeviceToHost, us));
    g_launches = launches;
    return LDPC_OK;
}

extern "C" ldpc_status ldpc_count_errors(const ldpc_code *code, int64_t n_frames, const uint32_t *hard_bits,
                                         const uint8_t *syndrome_ok, const int32_t *iterations_used,
                                         int64_t *counters, void *stream) {
    g_detail.clear();
    if (!code || !hard_bits || !syndrome_ok || !counters) return fail(LDPC_ERR_INVALID_ARG, "NULL argument");
    if (n_frames == 0) return LDPC_OK;
    DeviceGuard guard(code->device);
    const int wpf = (code->N + 31) / 32;
    cudaError_t e = count_errors_launch(n_frames, wpf, hard_bits, syndrome_ok, iterations_used,
                                        (unsigned long long *)counters, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(LDPC_ERR_CUDA, "count kernel: %s", cudaGetErrorString(e));
    return LDPC_OK;
}

extern "C" int32_t ldpc_last_launch_count(void) { return g_launches; }

extern "C" const char *ldpc_status_string(ldpc_status s) {
    switch (s) {
    case LDPC_OK: return "LDPC_OK";
    case LDPC_ERR_INVALID_ARG: return "LDPC_ERR_INVALID_ARG";
    case LDPC_ERR_INVALID_CODE: return "LDPC_ERR_INVALID_CODE";
    case LDPC_ERR_UNSUPPORTED: return "LDPC_ERR_UNSUPPORTED";
    case LDPC_ERR_CUDA: return "LDPC_ERR_CUDA";
    case LDPC_ERR_NO_MEMORY: return "LDPC_ERR_NO_MEMORY";
    }
    return "LDPC_ERR_UNKNOWN";
}

extern "C" const char *ldpc_last_error_detail(void) { return g_detail.c_str(); }

extern "C" int32_t ldpc_version(void) { return 100; }

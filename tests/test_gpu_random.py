"""Seeded random sweep: code shapes (QC with Z below / around / above one 128-thread
group, regular and irregular CSR codes, degree-1 and degree-2 columns), LLR types,
message formats, schedules, kernels (resident atom / batched, streaming pipe /
register), offsets, clamps and early stop -- every case bit-exact against the oracle
(integer LLRs).  Each case prints its parameters on failure (pytest ids)."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, gpu_decode  # noqa: E402


def _code(rng, i):
    kind = i % 4
    if kind == 0:
        mb = int(rng.integers(2, 7))
        nb = int(rng.integers(mb + 2, 3 * mb + 3))
        Z = int(rng.choice([5, 17, 31, 32, 64, 100, 127, 128, 129, 200]))
        w = rng.integers(1, min(mb, 4) + 1, nb).astype(np.int32)
        w[rng.integers(0, nb)] = min(mb, 2)
        return g.qc(mb, nb, Z, w, seed=int(rng.integers(1, 1 << 30)))
    if kind == 1:
        dv, dc = [(2, 4), (3, 6), (4, 8), (3, 5)][int(rng.integers(0, 4))]
        N = dc * int(rng.integers(6, 60))
        N -= N % dc
        return g.regular(N, dv, dc, seed=int(rng.integers(1, 1 << 30)), remove_4cycles=False)
    if kind == 2:                                  # info edges must fill every check equally
        M = 4 * int(rng.integers(3, 50))
        n_hi, w_hi = ((M // 2, 5), (M // 4, 7))[int(rng.integers(0, 2))]
        return g.dvbs2like(2 * M, M, n_hi, w_hi, 3, seed=int(rng.integers(1, 1 << 30)))
    M, N = int(rng.integers(3, 12)), int(rng.integers(8, 40))
    H = np.zeros((M, N), np.uint8)
    for m in range(M):                             # row degrees 2..8
        H[m, rng.choice(N, int(rng.integers(2, min(8, N) + 1)), replace=False)] = 1
    for n in range(N):                             # every column degree >= 1 (rows stay <= 8 if possible)
        if H[:, n].sum() == 0:
            rows = np.flatnonzero(H.sum(axis=1) < 8)
            H[rng.choice(rows) if len(rows) else rng.integers(0, M), n] = 1
    return g.from_dense(H, name="rand")


CASES = list(range(240))


@pytest.mark.parametrize("i", CASES)
def test_random_case(i):
    rng = np.random.default_rng(1000 + i)
    code = _code(rng, i)
    max_dc = int(np.max(np.diff(code.row_ptr)))
    if max_dc > 8:
        pytest.skip("integer paths support row degree <= 8")
    onebit = bool(rng.integers(0, 2))
    Q = int(rng.choice([31, 63, 127])) if onebit else int(rng.choice([63, 255, 511]))
    max_dv = int(np.max(np.bincount(code.col_idx, minlength=code.n_vars)))
    if 2 * Q * (max_dv + 2) > 32767:
        Q = 127
    lt, kind, frac = (P.LDPC_LLR_I8, g.LLR_I8, 2) if onebit and Q <= 127 and rng.integers(0, 2) else \
        (P.LDPC_LLR_I16, g.LLR_I16, 3)
    sched = [P.LDPC_SCHED_SINGLESCAN, P.LDPC_SCHED_SINGLESCAN, P.LDPC_SCHED_LAYERED,
             P.LDPC_SCHED_TWOSCAN][int(rng.integers(0, 4))]
    fmt = P.LDPC_MSG_1BIT if onebit else P.LDPC_MSG_COMPACT
    if sched == P.LDPC_SCHED_TWOSCAN:
        fmt = P.LDPC_MSG_COMPACT
    elif sched == P.LDPC_SCHED_SINGLESCAN and rng.integers(0, 3) == 0:
        fmt = P.LDPC_MSG_FULL                      # the §4 per-edge form (resident kernel only)
    env = [None, "stream", "batched", "stream-registers"][int(rng.integers(0, 4))]
    tuning = {None: None, "stream": {"path": P.LDPC_PATH_STREAM},
              "batched": {"path": P.LDPC_PATH_RESIDENT_BATCHED},
              "stream-registers": {"path": P.LDPC_PATH_STREAM, "stream_register_kernels": 1}}[env]
    K = int(rng.integers(1, 14))
    es = int(rng.integers(0, 2))
    beta = int(rng.integers(0, 3))
    F = int(rng.choice([1, 2, 3, 33, 64, 65, 130]))
    ebn0 = float(rng.uniform(0.5, 4.0))
    llr = g.llr(int(rng.integers(1, 1 << 30)), 0, F, code.n_vars, g.ebn0_to_sigma2(ebn0, max(code.rate, 0.2)),
                kind, frac, Q)
    # per-iteration beta_k / lambda_k on a third of the cases, from a separate
    # stream so the other parameters of each case stay as they were
    rs = np.random.default_rng(5000 + i)
    kw, okw = {}, {}
    if rs.integers(0, 3) == 0:
        okw["beta_sched"] = kw["offset_per_iter"] = [int(x) for x in rs.integers(0, 3, K)]
        if rs.integers(0, 2) == 0:
            okw["alpha_sched"] = kw["alpha_per_iter"] = [float(x) for x in rs.choice([1.0, 0.5, 0.75, 0.875], K)]
    params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, fmt, sched, tuning=tuning, **kw)
    try:
        post, hb, ok, it = gpu_decode(code, llr, params)
    except P.LdpcError as e:
        assert e.status == P.LDPC_ERR_UNSUPPORTED, str(e)
        pytest.skip(f"unsupported: {e}")
    engine = {P.LDPC_SCHED_SINGLESCAN: "compact", P.LDPC_SCHED_LAYERED: "layered",
              P.LDPC_SCHED_TWOSCAN: "twoscan"}[sched]
    ref = oracle.decode(code, llr.astype(np.int32), engine, "int", K, es, beta, Q, nthreads=NT, **okw)
    info = f"{code.name} N={code.n_vars} M={code.n_checks} sched={sched} env={env} K={K} es={es} beta={beta} Q={Q} " \
           f"F={F} fmt={fmt} lt={lt} schedules={okw}"
    np.testing.assert_array_equal(it, ref.iters, err_msg=info)
    np.testing.assert_array_equal(ok, ref.ok, err_msg=info)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post, err_msg=info)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits), err_msg=info)

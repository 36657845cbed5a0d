"""Seeded random sweep for fp32 LLRs: code shapes (QC, regular, DVB-S2-like, random CSR),
schedules (flooding on the pipelined / register streaming kernels, layered, two-scan),
variants, per-frame early stop.  Every case is bit-exact with the fp32 oracle: flooding
and two-scan sum posteriors exactly and round once (reading D28), layered updates in a
fixed order (reading D25)."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, assert_f32_exact, gpu_decode  # noqa: E402
from test_gpu_random import _code  # noqa: E402

CASES = list(range(120))


@pytest.mark.parametrize("i", CASES)
def test_random_f32_case(i):
    rng = np.random.default_rng(5000 + i)
    code = _code(rng, i)
    sched = [P.LDPC_SCHED_SINGLESCAN, P.LDPC_SCHED_LAYERED, P.LDPC_SCHED_TWOSCAN][i % 3]
    if sched != P.LDPC_SCHED_SINGLESCAN and int(np.max(np.diff(code.row_ptr))) > 8:
        pytest.skip("layered / two-scan kernels: row degree <= 8")
    tuning = {"stream_register_kernels": 1} if sched == P.LDPC_SCHED_SINGLESCAN and rng.integers(0, 2) else None
    K = int(rng.integers(1, 31))
    es = int(rng.integers(0, 2))
    if rng.integers(0, 2):
        variant, alpha, beta = P.LDPC_MINSUM_NORMALIZED, float(rng.choice([0.625, 0.75, 0.8, 1.0])), 0.0
    else:
        variant, alpha, beta = P.LDPC_MINSUM_OFFSET, 1.0, float(rng.choice([0.0, 0.125, 0.5]))
    F = int(rng.choice([1, 2, 31, 33, 64, 97]))
    llr = g.llr(int(rng.integers(1, 1 << 30)), 0, F, code.n_vars,
                g.ebn0_to_sigma2(float(rng.uniform(0.5, 4.0)), max(code.rate, 0.2)), g.LLR_F32)
    params = P.make_params(K, es, variant, 0, beta, alpha, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, sched,
                           tuning=tuning)
    try:
        post, hb, ok, it = gpu_decode(code, llr, params)
    except P.LdpcError as e:
        assert e.status == P.LDPC_ERR_UNSUPPORTED, str(e)
        pytest.skip(f"unsupported: {e}")
    engine = {P.LDPC_SCHED_SINGLESCAN: "compact", P.LDPC_SCHED_LAYERED: "layered",
              P.LDPC_SCHED_TWOSCAN: "twoscan"}[sched]
    ref = oracle.decode(code, llr, engine, "f32", K, es, beta=beta, alpha=alpha, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)

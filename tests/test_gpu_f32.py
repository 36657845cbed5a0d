"""fp32 LLRs (config 5's numeric form) on every fp32 path: bit-exact with the fp32 oracle
(reading D28: posterior sums exact and rounded once, so the GPU's atomic arrival order does
not matter), byte-identical from run to run and independent of batch composition, with
saturation at +-2^20 (D28) and -0.0 canonicalisation (D13) on load."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, assert_f32_exact, gpu_decode, small_codes  # noqa: E402


def _params(K, es, variant=P.LDPC_MINSUM_NORMALIZED, alpha=0.75, beta=0.0, sched=P.LDPC_SCHED_SINGLESCAN, **tn):
    return P.make_params(K, es, variant, 0, beta, alpha, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, sched,
                         tuning=tn or None)


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
@pytest.mark.parametrize("sched,engine", [(P.LDPC_SCHED_SINGLESCAN, "compact"), (P.LDPC_SCHED_TWOSCAN, "twoscan"),
                                          (P.LDPC_SCHED_LAYERED, "layered")], ids=["flood", "twoscan", "layered"])
def test_f32_small_codes_exact(code, sched, engine):
    """Several tiles and a ragged last tile, early stop on and off, both variants."""
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 70):
        llr = g.llr(300 + F, 0, F, code.n_vars, s2, g.LLR_F32)
        for variant, alpha, beta, es, K in ((P.LDPC_MINSUM_NORMALIZED, 0.75, 0.0, 0, 30),
                                            (P.LDPC_MINSUM_OFFSET, 1.0, 0.25, 1, 20)):
            post, hb, ok, it = gpu_decode(code, llr, _params(K, es, variant, alpha, beta, sched))
            ref = oracle.decode(code, llr, engine, "f32", K, es, beta=beta, alpha=alpha, nthreads=NT)
            assert_f32_exact(post, hb, ok, it, ref)


@pytest.mark.parametrize("es", [0, 1])
def test_f32_cfg2_code_mixed_convergence(es):
    """The cfg2 QC code at 2.0 dB: frames stop at different iterations (early stop), the
    rest oscillate for 30 iterations -- the frames whose fp32 sums drifted with the order of
    round 1's float atomics are now bit-exact."""
    code = g.CONFIGS[2].code()
    llr = g.llr(2222, 0, 200, code.n_vars, g.ebn0_to_sigma2(2.0, code.rate), g.LLR_F32)
    post, hb, ok, it = gpu_decode(code, llr, _params(30, es))
    ref = oracle.decode(code, llr, "compact", "f32", 30, es, alpha=0.75, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)
    if es:
        assert len(np.unique(ref.iters)) >= 3


def test_f32_run_to_run_and_batch_composition():
    """Two decodes of the same batch are byte-identical, and each frame's outputs do not
    depend on the other frames of its batch (same bits decoded 64 frames at a time)."""
    code = small_codes()[6]
    llr = g.llr(77, 0, 256, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_F32)
    p = _params(40, 0)
    a = gpu_decode(code, llr, p)
    b = gpu_decode(code, llr, p)
    parts = [gpu_decode(code, llr[i:i + 64], p) for i in range(0, 256, 64)]
    for x, y in zip(a, b):
        np.testing.assert_array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    for k in range(4):
        np.testing.assert_array_equal(np.concatenate([q[k] for q in parts]).view(np.uint8),
                                      np.asarray(a[k]).view(np.uint8))


def test_f32_extremes_saturation_and_negative_zero():
    """Channel values beyond 2^20 saturate (reading D28), -0.0 reads as +0.0 (D13), tiny
    values below the 2^-34 grid still give the right first-iteration signs (iteration 1
    reads the fp32 Z^(0) plane itself), and a noiseless high-SNR batch whose messages grow
    geometrically stays bit-exact through 60 iterations."""
    code = small_codes()[1]
    rng = np.random.default_rng(5)
    llr = g.llr(91, 0, 40, code.n_vars, 0.8, g.LLR_F32)
    llr[0, :7] = np.array([3e7, -5e9, -0.0, 1e-30, -1e-38, 2.0 ** 20, 7e-12], np.float32)
    llr[1] = np.float32(-0.0)
    llr[2] = rng.choice([1e-20, 1e-9, 3e-3], code.n_vars).astype(np.float32)
    for es in (0, 1):
        post, hb, ok, it = gpu_decode(code, llr, _params(12, es, P.LDPC_MINSUM_OFFSET, 1.0, 0.0))
        ref = oracle.decode(code, llr, "compact", "f32", 12, es, alpha=1.0, nthreads=NT)
        assert_f32_exact(post, hb, ok, it, ref)
    big = np.full((4, code.n_vars), 50.0, np.float32)
    post, hb, ok, it = gpu_decode(code, big, _params(60, 0, P.LDPC_MINSUM_OFFSET, 1.0, 0.0))
    ref = oracle.decode(code, big, "compact", "f32", 60, 0, alpha=1.0, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)
    assert np.max(np.abs(ref.post)) >= 2.0 ** 20          # the message saturation was reached


def test_f32_wide_rows_register_kernel():
    """Row degree 12 (> 8): the fp32 register kernel (the pipeline takes dc <= 8)."""
    code = g.regular(120, 6, 12, seed=2, remove_4cycles=False)
    llr = g.llr(4, 0, 40, code.n_vars, g.ebn0_to_sigma2(3.0, code.rate), g.LLR_F32)
    for es in (0, 1):
        post, hb, ok, it = gpu_decode(code, llr, _params(15, es))
        ref = oracle.decode(code, llr, "compact", "f32", 15, es, alpha=0.75, nthreads=NT)
        assert_f32_exact(post, hb, ok, it, ref)

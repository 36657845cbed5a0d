"""GPU two-scan baseline (LDPC_SCHED_TWOSCAN) against the CPU oracle's
two-scan engine (§3).

Integer LLRs: bit-exact posteriors, hard bits, flags and iteration counts -- the oracle's
two-scan is itself bit-exact with the compact single-scan (pinned in
tests/test_oracle.py), so these also show the GPU two-scan and single-scan agree.
fp32: bit-exact as well -- both sides evaluate Eq.(2)'s sums exactly and round once
(reading D28), so the GPU's extrinsic Z_n - L_mn (reading D24) equals the oracle's sum over
m' != m.
"""
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

TS = P.LDPC_SCHED_TWOSCAN


def assert_ts_int(code, llr, params, K, es, beta, Q):
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), "twoscan", "int", K, es, beta, Q, nthreads=NT)
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(ok, ref.ok)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))
    return post, hb, ok, it


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
def test_twoscan_small_codes_int(code):
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F, kind, frac, Q, lt in ((1, g.LLR_I16, 3, 511, P.LDPC_LLR_I16), (130, g.LLR_I16, 3, 511, P.LDPC_LLR_I16),
                                 (67, g.LLR_I8, 2, 127, P.LDPC_LLR_I8)):
        llr = g.llr(200 + F, 0, F, code.n_vars, sigma2, kind, frac, Q)
        for beta, es, K in ((1, 0, 12), (0, 1, 15), (2, 1, 5)):
            params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, P.LDPC_MSG_COMPACT, TS)
            assert_ts_int(code, llr, params, K, es, beta, Q)


@pytest.mark.parametrize("code", small_codes()[1:], ids=lambda c: c.name)
def test_twoscan_small_codes_f32(code):
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 33):
        llr = g.llr(7 + F, 0, F, code.n_vars, s2, g.LLR_F32)
        for variant, alpha, beta, es in ((P.LDPC_MINSUM_NORMALIZED, 0.75, 0.0, 0), (P.LDPC_MINSUM_OFFSET, 1.0, 0.25, 1)):
            params = P.make_params(10, es, variant, 0, beta, alpha, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, TS)
            post, hb, ok, it = gpu_decode(code, llr, params)
            ref = oracle.decode(code, llr, "twoscan", "f32", 10, es, beta=beta, alpha=alpha, nthreads=NT)
            assert_f32_exact(post, hb, ok, it, ref)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4])
def test_twoscan_configs_int(cfg_idx):
    """The BASELINE configs' codes and channels (parity subsets), two-scan schedule;
    also identical to the GPU single-scan decode of the same frames."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    F = min(cfg.parity_frames, 256)
    llr = cfg.llrs(code, 0, F)
    params = P.params_for_config(cfg, TS)
    post, hb, ok, it = assert_ts_int(code, llr, params, cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)
    p2, hb2, ok2, it2 = gpu_decode(code, llr, P.params_for_config(cfg))
    np.testing.assert_array_equal(post, p2)
    np.testing.assert_array_equal(it, it2)


def test_twoscan_cfg5_f32():
    cfg = g.CONFIGS[5]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 32)
    post, hb, ok, it = gpu_decode(code, llr, P.params_for_config(cfg, TS))
    ref = oracle.decode(code, llr, "twoscan", "f32", cfg.max_iter, 0, alpha=cfg.alpha, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)


def test_twoscan_unsupported():
    code = g.CONFIGS[1].code()
    from test_gpu_parity import decoder
    dec = decoder(code)
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(5, 0, P.LDPC_MINSUM_OFFSET, 1, 0, 1.0, 127, P.LDPC_LLR_I8, P.LDPC_MSG_1BIT, TS))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(5, 0, schedule=7))
    assert e.value.status == P.LDPC_ERR_INVALID_ARG

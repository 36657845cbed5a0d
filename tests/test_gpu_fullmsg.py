"""The §4 single-scan with stored per-edge messages (LDPC_MSG_FULL) on
the barrier-free resident kernel, against the oracle's per-edge single-scan engine
(``singlescan``) -- bit-exact, and identical to the compact form."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, decoder, gpu_decode, small_codes  # noqa: E402

FULL = P.LDPC_MSG_FULL


def assert_full(code, llr, params, K, es, beta, Q, **kw):
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), "singlescan", "int", K, es, beta, Q, nthreads=NT, **kw)
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(ok, ref.ok)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))
    return post, it


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
def test_full_small_codes(code):
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F, kind, frac, Q, lt in ((1, g.LLR_I16, 3, 511, P.LDPC_LLR_I16), (67, g.LLR_I16, 3, 511, P.LDPC_LLR_I16),
                                 (130, g.LLR_I8, 2, 127, P.LDPC_LLR_I8)):
        llr = g.llr(400 + F, 0, F, code.n_vars, s2, kind, frac, Q)
        for beta, es, K in ((1, 0, 12), (0, 1, 15), (2, 1, 5)):
            params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, FULL)
            assert_full(code, llr, params, K, es, beta, Q)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_full_configs_equal_compact(cfg_idx):
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 257)
    post, it = assert_full(code, llr, P.params_for_config(cfg, msg_format=FULL), cfg.max_iter, cfg.early_stop,
                           cfg.offset_raw, cfg.clamp)
    p2, hb2, ok2, it2 = gpu_decode(code, llr, P.params_for_config(cfg))
    np.testing.assert_array_equal(post, p2)
    np.testing.assert_array_equal(it, it2)


def test_full_schedules_and_normalized():
    code = small_codes()[4]
    llr = g.llr(77, 0, 40, code.n_vars, g.ebn0_to_sigma2(1.5, code.rate), g.LLR_I16, 3, 511)
    bs = [2, 1, 1, 0, 0, 0, 1, 0, 0, 0]
    al = [0.5, 0.75, 0.75, 1.0, 1.0, 0.875, 0.875, 1.0, 1.0, 1.0]
    params = P.make_params(10, 1, P.LDPC_MINSUM_OFFSET, 0, 0.0, 1.0, 511, P.LDPC_LLR_I16, FULL,
                           offset_per_iter=bs, alpha_per_iter=al)
    assert_full(code, llr, params, 10, 1, 0, 511, beta_sched=bs, alpha_sched=al)


def test_full_unsupported():
    dec = decoder(g.CONFIGS[4].code())                       # streaming-size code
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(64, P.params_for_config(g.CONFIGS[4], msg_format=FULL))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    dec = decoder(g.CONFIGS[2].code())
    with pytest.raises(P.LdpcError) as e:                    # layered keeps the compact state
        dec.workspace(64, P.params_for_config(g.CONFIGS[2], P.LDPC_SCHED_LAYERED, msg_format=FULL))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED


def test_full_unsupported_after_path_switch():
    """Requests that the planner moves off the barrier-free resident kernel after the format
    check -- per-iteration schedules longer than 64 iterations (streaming kernels), a forced
    streaming path, the batched resident kernel -- are rejected, never silently decoded with
    byte-wide magnitudes (round-1 advisor finding)."""
    code = g.CONFIGS[1].code()
    dec = decoder(code)
    long = P.make_params(70, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, FULL,
                         alpha_per_iter=[1.0] * 70)
    for params in (long,
                   P.make_params(5, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, FULL,
                                 tuning={"path": P.LDPC_PATH_STREAM}),
                   P.make_params(5, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, FULL,
                                 tuning={"path": P.LDPC_PATH_RESIDENT_BATCHED})):
        with pytest.raises(P.LdpcError) as e:
            dec.workspace(8, params)
        assert e.value.status == P.LDPC_ERR_UNSUPPORTED

"""GPU layered schedule (LDPC_SCHED_LAYERED, reading D25) against the
CPU oracle's layered engine: bit-exact posteriors, hard bits, syndrome flags and
iteration counts (integer LLRs, compact and 1-bit formats, early stop on and off; fp32
LLRs, where the in-place schedule makes the order of operations the oracle's)."""
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

LAY = P.LDPC_SCHED_LAYERED


def assert_lay(code, llr, params, K, es, beta, Q):
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), "layered", "int", K, es, beta, Q, nthreads=NT)
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(ok, ref.ok)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))
    return ref


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
@pytest.mark.parametrize("fmt", ["compact", "1bit"])
def test_layered_small_codes(code, fmt):
    Q = 511 if fmt == "compact" else 127
    kind, frac, lt = (g.LLR_I16, 3, P.LDPC_LLR_I16) if fmt == "compact" else (g.LLR_I8, 2, P.LDPC_LLR_I8)
    mf = P.LDPC_MSG_COMPACT if fmt == "compact" else P.LDPC_MSG_1BIT
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 2, 67, 130):
        llr = g.llr(300 + F, 0, F, code.n_vars, sigma2, kind, frac, Q)
        for beta, es, K in ((1, 0, 12), (0, 1, 15), (2, 1, 5)):
            params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, mf, LAY)
            assert_lay(code, llr, params, K, es, beta, Q)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_layered_configs(cfg_idx):
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 301)
    assert_lay(code, llr, P.params_for_config(cfg, LAY), cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)


def test_layered_mixed_convergence_cfg2_code():
    """2.25 dB on the cfg2 code: frames stop at different iterations; layered needs
    fewer iterations on average than flooding for the frames both decode."""
    cfg = g.CONFIGS[2]
    code = cfg.code()
    llr = g.llr(99, 0, 200, code.n_vars, g.ebn0_to_sigma2(2.25, code.rate), g.LLR_I16, 3, 511)
    ref = assert_lay(code, llr, P.params_for_config(cfg, LAY), 15, 1, 1, 511)
    post, hb, ok, it = gpu_decode(code, llr, P.params_for_config(cfg))
    both = (ok == 1) & (ref.ok == 1)
    assert both.sum() > 20
    assert ref.iters[both].mean() < it[both].mean()


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
@pytest.mark.parametrize("fmt", ["compact", "1bit", "f32"])
def test_layered_streaming_kernel_small_codes(code, fmt):
    """The streaming layered kernel (k_stream_layered.cuh: one warp per frame tile walking
    the rows in order), forced onto small codes with tuning.path = STREAM: bit-exact with the
    oracle's layered engine (D25) -- several tiles, a ragged last tile, early stop on and off."""
    if int(np.max(np.diff(code.row_ptr))) > 8:
        pytest.skip("row degree <= 8")
    tn = {"path": P.LDPC_PATH_STREAM}
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 70):
        for es, K in ((0, 9), (1, 14)):
            if fmt == "f32":
                llr = g.llr(800 + F, 0, F, code.n_vars, s2, g.LLR_F32)
                params = P.make_params(K, es, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32,
                                       P.LDPC_MSG_COMPACT, LAY, tuning=tn)
                post, hb, ok, it = gpu_decode(code, llr, params)
                ref = oracle.decode(code, llr, "layered", "f32", K, es, alpha=0.75, nthreads=NT)
                np.testing.assert_array_equal(it, ref.iters)
                np.testing.assert_array_equal(ok, ref.ok)
                np.testing.assert_array_equal(post.view(np.uint32), ref.post.astype(np.float32).view(np.uint32))
            else:
                Q, lt, gk, frac = (127, P.LDPC_LLR_I8, g.LLR_I8, 2) if fmt == "1bit" else (511, P.LDPC_LLR_I16, g.LLR_I16, 3)
                llr = g.llr(900 + F, 0, F, code.n_vars, s2, gk, frac, Q)
                params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, Q, lt,
                                       P.LDPC_MSG_1BIT if fmt == "1bit" else P.LDPC_MSG_COMPACT, LAY, tuning=tn)
                assert_lay(code, llr, params, K, es, 1, Q)
            assert P.ldpc_last_launch_count() > 1                    # the streaming layout


@pytest.mark.parametrize("cfg_idx", [4, 5])
def test_layered_long_codes(cfg_idx):
    """Configs 4 (int16) and 5 (fp32) codes, N = 64,800: the layered schedule runs on the
    streaming layered kernel (no longer UNSUPPORTED), bit-exact with the oracle on a few
    frames and iterations (the schedule is a chain of 32,400 dependent row updates per
    frame-iteration, so this is kept short), early stop on."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    s2 = g.ebn0_to_sigma2(1.5, code.rate)
    if cfg.llr_kind == g.LLR_F32:
        llr = g.llr(71, 0, 3, code.n_vars, s2, g.LLR_F32)
        params = P.make_params(4, 1, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                               LAY)
        post, hb, ok, it = gpu_decode(code, llr, params)
        ref = oracle.decode(code, llr, "layered", "f32", 4, 1, alpha=0.75, nthreads=NT)
        np.testing.assert_array_equal(it, ref.iters)
        np.testing.assert_array_equal(post.view(np.uint32), ref.post.astype(np.float32).view(np.uint32))
    else:
        llr = g.llr(72, 0, 3, code.n_vars, s2, g.LLR_I16, 3, 511)
        params = P.make_params(4, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, LAY)
        assert_lay(code, llr, params, 4, 1, 1, 511)


def test_layered_streaming_schedules():
    """Per-iteration lambda_k / beta_k on the streaming layered kernel
    (integer and fp32), bit-exact with the oracle's layered engine."""
    code = small_codes()[5]
    tn = {"path": P.LDPC_PATH_STREAM}
    K = 8
    bs = [2, 1, 1, 0, 0, 1, 0, 0]
    al = [0.5, 0.75, 0.75, 1.0, 0.875, 1.0, 0.75, 1.0]
    llr = g.llr(41, 0, 70, code.n_vars, g.ebn0_to_sigma2(1.5, code.rate), g.LLR_I16, 3, 511)
    params = P.make_params(K, 1, P.LDPC_MINSUM_OFFSET, 0, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, LAY,
                           offset_per_iter=bs, alpha_per_iter=al, tuning=tn)
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), "layered", "int", K, 1, 0, 511, nthreads=NT, beta_sched=bs,
                        alpha_sched=al)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(it, ref.iters)
    z = g.llr(42, 0, 40, code.n_vars, g.ebn0_to_sigma2(1.5, code.rate), g.LLR_F32)
    alf = np.linspace(0.6, 0.95, K).astype(np.float32)
    params = P.make_params(K, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, LAY,
                           alpha_per_iter=alf, tuning=tn)
    post, hb, ok, it = gpu_decode(code, z, params)
    ref = oracle.decode(code, z, "layered", "f32", K, 0, alpha=0.75, nthreads=NT, alpha_sched=alf.astype(np.float64))
    np.testing.assert_array_equal(post.view(np.uint32), ref.post.astype(np.float32).view(np.uint32))


@pytest.mark.parametrize("fmt", ["compact", "f32"])
def test_layered_streaming_messages(fmt):
    """Exit messages of the streaming layered kernel (ldpc_decode_batch_messages) against the
    oracle's layered trace of the last iteration (messages rebuilt from the compact state)."""
    code = small_codes()[6]
    tn = {"path": P.LDPC_PATH_STREAM}
    K = 7
    dec = decoder(code)
    if fmt == "f32":
        llr = g.llr(31, 0, 70, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_F32)
        params = P.make_params(K, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                               LAY, tuning=tn)
        ref = oracle.decode(code, llr, "layered", "f32", K, 0, alpha=0.75, trace=True, nthreads=NT)
    else:
        llr = g.llr(32, 0, 70, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_I16, 3, 511)
        params = P.make_params(K, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, LAY,
                               tuning=tn)
        ref = oracle.decode(code, llr.astype(np.int32), "layered", "int", K, 0, 1, 511, trace=True, nthreads=NT)
    out, msg = dec.decode_messages(torch.from_numpy(llr).cuda(), params)
    torch.cuda.synchronize()
    got = msg.cpu().numpy()
    if fmt == "f32":
        np.testing.assert_array_equal(got.view(np.uint32), ref.trace_msg[:, K - 1, :].astype(np.float32).view(np.uint32))
    else:
        np.testing.assert_array_equal(got.astype(np.int32), ref.trace_msg[:, K - 1, :])

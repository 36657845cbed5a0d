"""Message / state parity (BASELINE.json north star: "bit-exact ... messages, posteriors,
hard bits, iteration counts").  ldpc_decode_batch_messages exports the check messages at
exit, rebuilt on the GPU from each row's persistent compact state (A_m, B_m, ñ_m, s_mn;
P:306) -- compared element by element with the oracle's trace of the
last iteration (also rebuilt from its compact state), so a wrong A, B, sign or argmin
anywhere fails.  Integer int16 (compact and FULL per-edge), 1-bit (int8) and fp32; the
resident and streaming kernels and the two-scan baseline."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, decoder, small_codes  # noqa: E402


def gpu_messages(code, llr, params):
    dec = decoder(code)
    out, msg = dec.decode_messages(torch.from_numpy(np.ascontiguousarray(llr)).cuda(), params)
    torch.cuda.synchronize()
    return (out.posteriors.cpu().numpy(), out.iterations.cpu().numpy(), msg.cpu().numpy())


def check(code, llr, params, engine, mode, K, es=0, beta=0, Q=0, alpha=1.0, frames=None):
    post, it, msg = gpu_messages(code, llr, params)
    sel = np.arange(llr.shape[0]) if frames is None else np.asarray(frames)
    z = llr[sel] if mode == "f32" else llr[sel].astype(np.int32)
    ref = oracle.decode(code, z, engine, mode, K, es, beta, Q, alpha=alpha, trace=True, nthreads=NT)
    np.testing.assert_array_equal(it[sel], ref.iters)
    full = ref.iters == K                                   # messages are defined for these frames
    assert full.any()
    want = ref.trace_msg[full, K - 1, :]
    got = msg[sel][full]
    if mode == "f32":
        np.testing.assert_array_equal(got.view(np.uint32), want.astype(np.float32).view(np.uint32))
        np.testing.assert_array_equal(post[sel].view(np.uint32), ref.post.astype(np.float32).view(np.uint32))
    else:
        np.testing.assert_array_equal(got.astype(np.int32), want)
        np.testing.assert_array_equal(post[sel].astype(np.int32), ref.post)
    return ref


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
@pytest.mark.parametrize("kind", ["compact", "1bit", "full", "stream", "stream-1bit", "twoscan"])
def test_messages_small_codes_int(code, kind):
    fmt = {"1bit": P.LDPC_MSG_1BIT, "stream-1bit": P.LDPC_MSG_1BIT, "full": P.LDPC_MSG_FULL}.get(kind, P.LDPC_MSG_COMPACT)
    sched = P.LDPC_SCHED_TWOSCAN if kind == "twoscan" else P.LDPC_SCHED_SINGLESCAN
    tuning = {"path": P.LDPC_PATH_STREAM} if kind.startswith("stream") else None
    engine = {"full": "singlescan", "twoscan": "twoscan"}.get(kind, "compact")
    onebit = fmt == P.LDPC_MSG_1BIT
    Q, lt, gk, frac = (127, P.LDPC_LLR_I8, g.LLR_I8, 2) if onebit else (511, P.LDPC_LLR_I16, g.LLR_I16, 3)
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 67):
        llr = g.llr(600 + F, 0, F, code.n_vars, s2, gk, frac, Q)
        for beta, es, K in ((1, 0, 9), (0, 1, 12)):
            params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, fmt, sched, tuning=tuning)
            check(code, llr, params, engine, "int", K, es, beta, Q) if es == 0 else _check_es(code, llr, params,
                                                                                             engine, K, beta, Q)


def _check_es(code, llr, params, engine, K, beta, Q):
    """Early stop on: only frames that ran all K iterations carry defined messages."""
    post, it, msg = gpu_messages(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), engine, "int", K, 1, beta, Q, trace=True, nthreads=NT)
    np.testing.assert_array_equal(it, ref.iters)
    full = ref.iters == K
    np.testing.assert_array_equal(msg[full].astype(np.int32), ref.trace_msg[full, K - 1, :])


@pytest.mark.parametrize("code", small_codes()[1:], ids=lambda c: c.name)
@pytest.mark.parametrize("sched,engine", [(P.LDPC_SCHED_SINGLESCAN, "compact"), (P.LDPC_SCHED_TWOSCAN, "twoscan")],
                         ids=["flood", "twoscan"])
def test_messages_small_codes_f32(code, sched, engine):
    llr = g.llr(71, 0, 40, code.n_vars, g.ebn0_to_sigma2(1.5, max(code.rate, 0.3)), g.LLR_F32)
    for variant, alpha, beta in ((P.LDPC_MINSUM_NORMALIZED, 0.75, 0.0), (P.LDPC_MINSUM_OFFSET, 1.0, 0.25)):
        params = P.make_params(14, 0, variant, 0, beta, alpha, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT, sched)
        check(code, llr, params, engine, "f32", 14, 0, beta, 0, alpha)


def test_messages_cfg1_full_batch_sampled():
    """Config 1 at its full batch (1024 frames, the bench launch): sampled frames' messages."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    llr = cfg.llrs(code, 0, cfg.frames)
    picks = np.unique(np.r_[0, 1, 511, 512, cfg.frames - 1, np.linspace(0, cfg.frames - 1, 20).astype(int)])
    check(code, llr, P.params_for_config(cfg), "compact", "int", cfg.max_iter, 0, cfg.offset_raw, cfg.clamp,
          frames=picks)


def test_messages_cfg3_1bit():
    """Config 3 (1-bit messages, int8 LLRs, 30 iterations): 2048 frames decoded, sampled
    frames across several 32-frame words compared."""
    cfg = g.CONFIGS[3]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 2048)
    picks = np.r_[0:4, 31:34, 1000:1003, 2044:2048]
    check(code, llr, P.params_for_config(cfg), "compact", "int", cfg.max_iter, 0, cfg.offset_raw, cfg.clamp,
          frames=picks)


@pytest.mark.parametrize("cfg_idx", [4, 5])
def test_messages_long_codes(cfg_idx):
    """Configs 4 (int16) and 5 (fp32) on the streaming kernels, 130 frames decoded (3 tiles,
    ragged), 4 frames compared (the oracle's trace of 50 iterations x 226,799 edges)."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 130)
    picks = [0, 63, 64, 129]
    if cfg.llr_kind == g.LLR_F32:
        check(code, llr, P.params_for_config(cfg), "compact", "f32", cfg.max_iter, 0, 0, 0, cfg.alpha, frames=picks)
    else:
        check(code, llr, P.params_for_config(cfg), "compact", "int", cfg.max_iter, 0, cfg.offset_raw, cfg.clamp,
              frames=picks)


def test_messages_unsupported():
    code = g.CONFIGS[1].code()
    llr = torch.zeros((4, code.n_vars), dtype=torch.int16, device="cuda")
    dec = decoder(code)
    for params in (P.params_for_config(g.CONFIGS[1], P.LDPC_SCHED_LAYERED),
                   P.set_tuning(P.params_for_config(g.CONFIGS[1]), {"path": P.LDPC_PATH_RESIDENT_BATCHED})):
        with pytest.raises(P.LdpcError) as e:
            dec.decode_messages(llr, params)
        assert e.value.status == P.LDPC_ERR_UNSUPPORTED


@pytest.mark.parametrize("i", list(range(80)))
def test_messages_random(i):
    """Seeded random sweep of the message export: code shapes of tests/test_gpu_random.py,
    integer (compact / 1-bit / FULL; resident, streaming pipeline, streaming register
    kernels) and fp32 (flooding, two-scan), fixed iteration counts."""
    from test_gpu_random import _code
    rng = np.random.default_rng(7000 + i)
    code = _code(rng, i)
    if int(np.max(np.diff(code.row_ptr))) > 8:
        pytest.skip("row degree > 8")
    K = int(rng.integers(1, 16))
    F = int(rng.choice([1, 3, 64, 65]))
    s2 = g.ebn0_to_sigma2(float(rng.uniform(0.5, 3.5)), max(code.rate, 0.2))
    kind = ["compact", "1bit", "full", "stream", "stream-reg", "f32", "f32-ts", "ts"][i % 8]
    tuning = {"stream": {"path": P.LDPC_PATH_STREAM},
              "stream-reg": {"path": P.LDPC_PATH_STREAM, "stream_register_kernels": 1}}.get(kind)
    try:
        if kind.startswith("f32"):
            llr = g.llr(int(rng.integers(1, 1 << 30)), 0, F, code.n_vars, s2, g.LLR_F32)
            sched, engine = (P.LDPC_SCHED_TWOSCAN, "twoscan") if kind == "f32-ts" else (P.LDPC_SCHED_SINGLESCAN, "compact")
            params = P.make_params(K, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                                   sched)
            check(code, llr, params, engine, "f32", K, 0, 0, 0, 0.75)
        else:
            onebit = kind == "1bit"
            Q, lt, gk, frac = (127, P.LDPC_LLR_I8, g.LLR_I8, 2) if onebit else (511, P.LDPC_LLR_I16, g.LLR_I16, 3)
            max_dv = int(np.max(np.bincount(code.col_idx, minlength=code.n_vars)))
            if 2 * Q * (max_dv + 2) > 32767:
                Q = 127
            llr = g.llr(int(rng.integers(1, 1 << 30)), 0, F, code.n_vars, s2, gk, frac, Q)
            fmt = {"1bit": P.LDPC_MSG_1BIT, "full": P.LDPC_MSG_FULL}.get(kind, P.LDPC_MSG_COMPACT)
            sched = P.LDPC_SCHED_TWOSCAN if kind == "ts" else P.LDPC_SCHED_SINGLESCAN
            engine = {"full": "singlescan", "ts": "twoscan"}.get(kind, "compact")
            beta = int(rng.integers(0, 3))
            params = P.make_params(K, 0, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, lt, fmt, sched, tuning=tuning)
            check(code, llr, params, engine, "int", K, 0, beta, Q)
    except P.LdpcError as e:
        assert e.status == P.LDPC_ERR_UNSUPPORTED, str(e)
        pytest.skip(f"unsupported: {e}")

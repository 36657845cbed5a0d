"""Per-iteration lambda_k / beta_k schedules and integer
normalized min-sum with a dyadic lambda (reading D27) -- SURVEY.md §8(f3) -- on every
GPU path, against the CPU oracle with the same schedules: bit-exact for integer LLRs and
for fp32 (reading D28)."""
import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402
from test_gpu_parity import NT, assert_f32_exact, decoder, gpu_decode, small_codes  # noqa: E402

K = 14
BETAS = [3, 2, 2, 1, 1, 1, 0, 0, 0, 1, 1, 0, 0, 0]
ALPHAS = [0.5, 0.625, 0.75, 0.75, 0.875, 0.875, 1.0, 1.0, 0.75, 0.75, 1.0, 1.0, 0.5, 1.0]


def run_int(code, llr, Q, lt, fmt, engine, es, sched, tuning=None, **kw):
    params = P.make_params(K, es, kw.get("variant", P.LDPC_MINSUM_OFFSET), kw.get("beta", 0), 0.0,
                           kw.get("alpha", 1.0), Q, lt, fmt, sched, offset_per_iter=kw.get("bs"),
                           alpha_per_iter=kw.get("al"), tuning=tuning or None)
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), engine, "int", K, es, kw.get("beta", 0), Q,
                        alpha=kw.get("alpha", 1.0), nthreads=NT, beta_sched=kw.get("bs"), alpha_sched=kw.get("al"))
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))
    np.testing.assert_array_equal(ok, ref.ok)


PATHS = [  # (schedule, oracle engine, plan overrides)
    ("flood-atom", P.LDPC_SCHED_SINGLESCAN, "compact", {}),
    ("flood-batched", P.LDPC_SCHED_SINGLESCAN, "compact", {"path": P.LDPC_PATH_RESIDENT_BATCHED}),
    ("flood-stream", P.LDPC_SCHED_SINGLESCAN, "compact", {"path": P.LDPC_PATH_STREAM}),
    ("layered", P.LDPC_SCHED_LAYERED, "layered", {}),
    ("twoscan", P.LDPC_SCHED_TWOSCAN, "twoscan", {}),
]


@pytest.mark.parametrize("path", PATHS, ids=lambda p: p[0])
@pytest.mark.parametrize("code", [small_codes()[i] for i in (1, 3, 4, 5)], ids=lambda c: c.name)
def test_int_schedules_and_normalized(path, code):
    name, sched, engine, env = path
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    llr = g.llr(51, 0, 67, code.n_vars, s2, g.LLR_I16, 3, 511)
    # constant dyadic lambda = 3/4 (normalized, integer), with and without an offset
    run_int(code, llr, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, engine, 1, sched, env,
            variant=P.LDPC_MINSUM_NORMALIZED, alpha=0.75)
    run_int(code, llr, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, engine, 0, sched, env,
            variant=P.LDPC_MINSUM_NORMALIZED, alpha=0.75, beta=1)
    # per-iteration beta_k and lambda_k
    run_int(code, llr, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, engine, 1, sched, env, bs=BETAS, al=ALPHAS)
    if sched != P.LDPC_SCHED_TWOSCAN:   # 1-bit messages (int8, Q = 127 = b = 8 bits)
        z8 = g.llr(52, 0, 33, code.n_vars, s2, g.LLR_I8, 2, 127)
        run_int(code, z8, 127, P.LDPC_LLR_I8, P.LDPC_MSG_1BIT, engine, 0, sched, env, bs=BETAS, al=ALPHAS)


@pytest.mark.parametrize("cfg_idx", [1, 2])
def test_config_codes_normalized_int(cfg_idx):
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 128)
    run_int(code, llr, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, "compact", cfg.early_stop, P.LDPC_SCHED_SINGLESCAN,
            variant=P.LDPC_MINSUM_NORMALIZED, alpha=0.75, beta=0)


def test_long_schedule_falls_back_to_streaming():
    """Schedules longer than the resident kernels' table (64) run on the streaming kernels."""
    code = small_codes()[3]
    llr = g.llr(53, 0, 40, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_I16, 3, 511)
    KK = 70
    bs = [i % 3 for i in range(KK)]
    params = P.make_params(KK, 0, P.LDPC_MINSUM_OFFSET, 0, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT,
                           offset_per_iter=bs)
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr.astype(np.int32), "compact", "int", KK, 0, 0, 511, nthreads=NT, beta_sched=bs)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)


def test_f32_schedules():
    cfg = g.CONFIGS[5]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 32)
    al = np.linspace(0.6, 0.9, cfg.max_iter).astype(np.float32)
    for sched, engine in ((P.LDPC_SCHED_SINGLESCAN, "compact"), (P.LDPC_SCHED_TWOSCAN, "twoscan")):
        params = P.make_params(cfg.max_iter, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32,
                               P.LDPC_MSG_COMPACT, sched, alpha_per_iter=al)
        post, hb, ok, it = gpu_decode(code, llr, params)
        ref = oracle.decode(code, llr, engine, "f32", cfg.max_iter, 0, alpha=0.75, nthreads=NT,
                            alpha_sched=al.astype(np.float64))
        assert_f32_exact(post, hb, ok, it, ref)
    small = small_codes()[1]
    z = g.llr(54, 0, 33, small.n_vars, g.ebn0_to_sigma2(1.5, small.rate), g.LLR_F32)
    bf = np.array([0.5, 0.5, 0.25, 0.25, 0.125, 0, 0, 0, 0, 0], np.float32)
    params = P.make_params(10, 1, P.LDPC_MINSUM_OFFSET, 0, 0.25, 1.0, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                           offset_f_per_iter=bf)
    post, hb, ok, it = gpu_decode(small, z, params)
    ref = oracle.decode(small, z, "compact", "f32", 10, 1, beta=0.25, nthreads=NT, beta_sched=bf.astype(np.float64))
    assert_f32_exact(post, hb, ok, it, ref)


def test_schedule_errors():
    code = g.CONFIGS[1].code()
    dec = decoder(code)
    with pytest.raises(P.LdpcError) as e:   # lambda = 0.7 is not dyadic
        dec.workspace(8, P.make_params(5, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.7, 511, P.LDPC_LLR_I16))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(3, 0, alpha_per_iter=[1.0, 0.0, 1.0]))
    assert e.value.status == P.LDPC_ERR_INVALID_ARG
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(3, 0, offset_per_iter=[1, -1, 0]))
    assert e.value.status == P.LDPC_ERR_INVALID_ARG

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer paths (int16 compact, int8 1-bit): bit-exact posteriors, hard bits,
syndrome flags and iteration counts (BASELINE.json north star).  fp32 path: bit-exact
as well -- both sides sum posteriors exactly and round once (reading D28) -- and, as the
north star's bar, within |dL| <= 1e-4 (1 + |L|) of the float64 oracle with hard bits
differing only where |L| < 1e-3.  Oracle inputs are the generator's bytes (ldpcgen),
never the GPU's.
"""
import os

import numpy as np
import pytest

import ldpcgen as g
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_cs_0609090_b200 as P  # noqa: E402

NT = max(1, min(64, os.cpu_count() or 1))
_DECODERS = {}


def decoder(code):
    key = id(code)
    if key not in _DECODERS:
        _DECODERS[key] = (code, P.Decoder(code, 0))
    return _DECODERS[key][1]


def tuned(params, **kw):
    """params with plan overrides (include/ldpc.h ldpc_tuning), e.g. path=P.LDPC_PATH_STREAM."""
    return P.set_tuning(params, kw)


def gpu_decode(code, llr, params, posteriors=True):
    dec = decoder(code)
    t = torch.from_numpy(np.ascontiguousarray(llr)).cuda()
    out = dec.decode(t, params, posteriors=posteriors)
    torch.cuda.synchronize()
    hb = out.hard_bits.cpu().numpy().view(np.uint32)
    post = out.posteriors.cpu().numpy() if out.posteriors is not None else None
    return post, hb, out.syndrome_ok.cpu().numpy(), out.iterations.cpu().numpy()


def oracle_decode_int(code, llr, K, es, beta, Q, frames=None):
    z = llr if frames is None else llr[frames]
    return oracle.decode(code, z.astype(np.int32), "compact", "int", K, es, beta, Q, nthreads=NT)


def assert_int_parity(code, llr, params, K, es, beta, Q, frames=None):
    post, hb, ok, it = gpu_decode(code, llr, params)
    sel = slice(None) if frames is None else frames
    ref = oracle_decode_int(code, llr, K, es, beta, Q, frames)
    np.testing.assert_array_equal(it[sel], ref.iters)
    np.testing.assert_array_equal(ok[sel], ref.ok)
    np.testing.assert_array_equal(post[sel].astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb[sel], oracle.pack_bits(ref.bits))
    return ref


def small_codes():
    return [
        g.from_dense([[1, 1, 0], [0, 1, 1]], name="toy"),
        g.regular(96, 3, 6, seed=5),
        g.regular(48, 3, 6, seed=9, remove_4cycles=False),
        g.qc(4, 8, 7, np.array([2, 3, 2, 3, 2, 2, 3, 2], np.int32), seed=3),
        g.qc(6, 12, 37, np.array([3, 4] * 6, np.int32), seed=8),
        g.dvbs2like(64, 32, 16, 5, 3, seed=4),
        g.dvbs2like(600, 300, 120, 8, 3, seed=6),
    ]


@pytest.mark.parametrize("code", small_codes(), ids=lambda c: c.name)
@pytest.mark.parametrize("force_stream", [False, True])
@pytest.mark.parametrize("fmt", ["compact", "1bit"])
def test_small_codes_int(code, force_stream, fmt):
    Q = 511 if fmt == "compact" else 127
    kind, frac = (g.LLR_I16, 3) if fmt == "compact" else (g.LLR_I8, 2)
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 2, 67, 130):                       # odd / ragged batches
        llr = g.llr(100 + F, 0, F, code.n_vars, sigma2, kind, frac, Q)
        for beta, es, K in ((1, 0, 12), (0, 1, 15), (2, 1, 5)):
            params = P.make_params(K, es, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q,
                                   P.LDPC_LLR_I16 if kind == g.LLR_I16 else P.LDPC_LLR_I8,
                                   P.LDPC_MSG_COMPACT if fmt == "compact" else P.LDPC_MSG_1BIT)
            if force_stream:
                tuned(params, path=P.LDPC_PATH_STREAM)
            assert_int_parity(code, llr, params, K, es, beta, Q)


def _cfg_params(cfg):
    return P.params_for_config(cfg)


def test_cfg1_all_frames():
    """Config 1: (3,6)-regular N=1008, 2.5 dB, offset 1, 20 iterations, all 1024 frames."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    llr = cfg.llrs(code, 0, cfg.frames)
    assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)


def test_cfg2_parity_subset_and_early_stop():
    """Config 2 (QC DTMB shape, <=15 iterations, early stop) on 1024 frames at 1.5 dB,
    plus 512 frames at 2.25 dB where early stop fires at spread-out iterations."""
    cfg = g.CONFIGS[2]
    code = cfg.code()
    llr = cfg.llrs(code, 0, cfg.parity_frames)
    assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, 1, cfg.offset_raw, cfg.clamp)
    s2 = g.ebn0_to_sigma2(2.25, code.rate)
    llr = g.llr(cfg.noise_seed + 77, 0, 512, code.n_vars, s2, g.LLR_I16, 3, 511)
    ref = assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, 1, cfg.offset_raw, cfg.clamp)
    assert len(np.unique(ref.iters)) >= 4 and ref.ok.mean() > 0.3      # early stop really exercised


def test_cfg3_parity_subset():
    """Config 3: 1-bit messages, int8 Q2 LLRs, 30 iterations (2048-frame subset, SURVEY
    §8(d): 64 whole 32-frame sign words)."""
    cfg = g.CONFIGS[3]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 2048)
    assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, 0, cfg.offset_raw, cfg.clamp)


def test_cfg4_parity_subset():
    """Config 4: DVB-S2 shape N=64800, 50 iterations, 64 frames (streaming kernels)."""
    cfg = g.CONFIGS[4]
    code = cfg.code()
    llr = cfg.llrs(code, 0, cfg.parity_frames)
    assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, 0, cfg.offset_raw, cfg.clamp)


def _assert_f32_parity(post, hb, ok, ref_post):
    """The north star's fp32 bar (used against the float64 oracle)."""
    scale = 1.0 + np.abs(ref_post)
    assert np.max(np.abs(post.astype(np.float64) - ref_post) / scale) <= 1e-4
    bits = (post <= 0).astype(np.uint8)
    ref_bits = (ref_post <= 0).astype(np.uint8)
    diff = bits != ref_bits
    assert np.all(np.abs(ref_post[diff]) < 1e-3)


def assert_f32_exact(post, hb, ok, it, ref):
    """fp32 GPU vs the fp32 oracle: identical bits (reading D28 makes both order-free)."""
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(ok, ref.ok)
    np.testing.assert_array_equal(post.view(np.uint32), ref.post.astype(np.float32).view(np.uint32))
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))


def test_cfg5_parity_subset():
    """Config 5: fp32 normalized (alpha 0.75), 50 iterations, 64 frames: bit-exact with the
    fp32 oracle, within the BJ tolerance of the float64 oracle, and byte-identical run to run."""
    cfg = g.CONFIGS[5]
    code = cfg.code()
    llr = cfg.llrs(code, 0, cfg.parity_frames)
    post, hb, ok, it = gpu_decode(code, llr, _cfg_params(cfg))
    ref = oracle.decode(code, llr, "compact", "f32", cfg.max_iter, 0, alpha=cfg.alpha, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)
    ref64 = oracle.decode(code, llr.astype(np.float64), "compact", "f64", cfg.max_iter, 0, alpha=cfg.alpha,
                          nthreads=NT)
    _assert_f32_parity(post, hb, ok, ref64.post)
    again = gpu_decode(code, llr, _cfg_params(cfg))
    np.testing.assert_array_equal(again[0].view(np.uint32), post.view(np.uint32))


@pytest.mark.parametrize("code", small_codes()[1:], ids=lambda c: c.name)
def test_small_codes_f32(code):
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (1, 33):
        llr = g.llr(5 + F, 0, F, code.n_vars, s2, g.LLR_F32)
        for variant, alpha, beta, es in ((P.LDPC_MINSUM_NORMALIZED, 0.75, 0.0, 0), (P.LDPC_MINSUM_OFFSET, 1.0, 0.25, 1)):
            for reg in (0, 1):                    # cp.async row pipeline / register kernels
                params = P.make_params(25, es, variant, 0, beta, alpha, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                                       tuning={"stream_register_kernels": reg})
                post, hb, ok, it = gpu_decode(code, llr, params)
                ref = oracle.decode(code, llr, "compact", "f32", 25, es, beta=beta, alpha=alpha, nthreads=NT)
                assert_f32_exact(post, hb, ok, it, ref)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4, 5])
def test_full_size_sampled_frames(cfg_idx):
    """At BASELINE.json's full batch size (the launch bench.py times), sampled frames
    (first, last, and spread) match the oracle decoding them one by one."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    F = cfg.frames
    llr = cfg.llrs(code, 0, F)
    post, hb, ok, it = gpu_decode(code, llr, _cfg_params(cfg))
    picks = np.unique(np.r_[0, 1, F - 2, F - 1, np.linspace(0, F - 1, 12).astype(int)])
    if cfg.llr_kind == g.LLR_F32:
        ref = oracle.decode(code, llr[picks], "compact", "f32", cfg.max_iter, 0, alpha=cfg.alpha, nthreads=NT)
        assert_f32_exact(post[picks], hb[picks], ok[picks], it[picks], ref)
    else:
        ref = oracle_decode_int(code, llr, cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp, picks)
        np.testing.assert_array_equal(post[picks].astype(np.int32), ref.post)
        np.testing.assert_array_equal(hb[picks], oracle.pack_bits(ref.bits))
        np.testing.assert_array_equal(ok[picks], ref.ok)
        np.testing.assert_array_equal(it[picks], ref.iters)
    # properties that hold at any size: converged frames are codewords; iterations within cap
    conv = ok == 1
    assert np.all((it >= 0) & (it <= cfg.max_iter))
    H_rows = [code.col_idx[code.row_ptr[m]:code.row_ptr[m + 1]] for m in range(0, code.n_checks, 97)]
    bits = np.unpackbits(hb[conv].view(np.uint8), axis=1, bitorder="little")[:, :code.n_vars]
    for r in H_rows:
        assert np.all(bits[:, r].sum(axis=1) % 2 == 0)


def test_noiseless_and_edge_cases():
    code = g.CONFIGS[2].code()
    params = P.make_params(15, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
    llr = np.full((5, code.n_vars), 40, np.int16)
    post, hb, ok, it = gpu_decode(code, llr, params)
    assert np.all(it == 0) and np.all(ok == 1) and np.all(hb == 0) and np.all(post == 40)
    # max_iter = 1
    cfg = g.CONFIGS[1]
    c1 = cfg.code()
    z = cfg.llrs(c1, 0, 9)
    p1 = P.make_params(1, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
    assert_int_parity(c1, z, p1, 1, 0, 1, 511)
    # out-of-range channel LLRs are saturated to +-Q on load
    zb = z.copy()
    zb[:, :5] = 3000
    post, hb, ok, it = gpu_decode(c1, zb, p1)
    ref = oracle_decode_int(c1, np.clip(zb, -511, 511), 1, 0, 1, 511)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    # n_frames = 0 is a no-op
    dec = decoder(c1)
    ws, nb = dec.workspace(0, p1)
    P.ldpc_decode_batch(dec.handle, p1, 0, 0, 0, 0, 0, 0, 0, 0, torch.cuda.current_stream().cuda_stream)


def test_unsupported_requests():
    c1 = g.CONFIGS[1].code()
    dec = decoder(c1)
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(5, 0, P.LDPC_MINSUM_OFFSET, 1, 0, 1.0, 600, P.LDPC_LLR_I16, P.LDPC_MSG_1BIT))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(5, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0, 0.7, 0, P.LDPC_LLR_I16))   # not dyadic
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(8, P.make_params(0, 0))
    assert e.value.status == P.LDPC_ERR_INVALID_ARG
    for bad in ({"resident_fixed_bases": 1}, {"resident_fixed_bases": -2}, {"resident_threads": 48},
                {"host_streams": 5}, {"path": 7}):
        with pytest.raises(P.LdpcError) as e:
            dec.workspace(8, P.make_params(5, 1, P.LDPC_MINSUM_OFFSET, 1, tuning=bad))
        assert e.value.status == P.LDPC_ERR_INVALID_ARG, bad
    # frame counts: int32 frame indices on the device; the size query alone (no allocation)
    params = _cfg_params(g.CONFIGS[1])
    assert P.ldpc_decode_workspace_size(dec.handle, 2**31 - 1, params) > 0
    for bad, status in ((2**31, P.LDPC_ERR_UNSUPPORTED), (-1, P.LDPC_ERR_INVALID_ARG)):
        with pytest.raises(P.LdpcError) as e:
            P.ldpc_decode_workspace_size(dec.handle, bad, params)
        assert e.value.status == status


def test_host_api_matches_device_api_and_counters():
    cfg = g.CONFIGS[2]
    code = cfg.code()
    F = 4100
    llr = cfg.llrs(code, 0, F)
    params = _cfg_params(cfg)
    post, hb, ok, it = gpu_decode(code, llr, params)
    dec = decoder(code)
    lh = torch.from_numpy(llr).pin_memory()
    hbh = torch.empty((F, dec.wpf), dtype=torch.int32).pin_memory()
    okh = torch.empty(F, dtype=torch.uint8).pin_memory()
    ith = torch.empty(F, dtype=torch.int32).pin_memory()
    ph = torch.empty((F, code.n_vars), dtype=torch.int16).pin_memory()
    dec.decode_host(lh, params, hbh, okh, ith, ph)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hbh.numpy().view(np.uint32), hb)
    np.testing.assert_array_equal(okh.numpy(), ok)
    np.testing.assert_array_equal(ith.numpy(), it)
    np.testing.assert_array_equal(ph.numpy(), post)
    # error counters (all-zero codeword, reading D14)
    out = dec.decode(torch.from_numpy(llr).cuda(), params)
    cnt = dec.count_errors(out).cpu().numpy()
    nbits = np.array([bin(int(x)).count("1") for x in hb.ravel()]).reshape(hb.shape).sum(axis=1)
    want = [nbits.sum(), (nbits > 0).sum(), ((nbits > 0) & (ok == 1)).sum(), (ok == 0).sum(), it.sum()]
    np.testing.assert_array_equal(cnt, want)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", ["pinned", "pageable"])
def test_host_api_output_modes(cfg_idx, mode):
    """ldpc_decode_batch_host with pinned and pageable host buffers, resident (cfg1-3) and
    streaming (cfg4) kernels, a partial last chunk and the optional outputs omitted:
    identical results to the device API."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    F = {1: 1100, 2: 1300, 3: 1100, 4: 150}[cfg_idx]
    llr = cfg.llrs(code, 0, F)
    params = _cfg_params(cfg)
    post, hb, ok, it = gpu_decode(code, llr, params)
    dec = decoder(code)

    def buf(t):
        return t if mode == "pageable" else t.pin_memory()

    lh = buf(torch.from_numpy(llr))
    hbh = buf(torch.full((F, dec.wpf), -1, dtype=torch.int32))
    okh = buf(torch.full((F,), 7, dtype=torch.uint8))
    ith = buf(torch.full((F,), -1, dtype=torch.int32))
    ph = buf(torch.full((F, code.n_vars), 12345, dtype=torch.int16))
    dec.decode_host(lh, params, hbh, okh, ith, ph)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hbh.numpy().view(np.uint32), hb)
    np.testing.assert_array_equal(okh.numpy(), ok)
    np.testing.assert_array_equal(ith.numpy(), it)
    np.testing.assert_array_equal(ph.numpy(), post)
    # optional outputs omitted
    hbh.fill_(-1)
    dec.decode_host(lh, params, hbh, okh)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hbh.numpy().view(np.uint32), hb)


def test_batch_composition_invariance():
    """Per-frame outputs do not depend on how frames are batched (the analog of
    decoding a global frame range on 1 or on W GPUs)."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 256)
    params = _cfg_params(cfg)
    full = gpu_decode(code, llr, params)
    parts = [gpu_decode(code, llr[a:a + 64], params) for a in range(0, 256, 64)]
    for i in range(4):
        np.testing.assert_array_equal(np.concatenate([p[i] for p in parts]), full[i])
    again = gpu_decode(code, llr, params)
    for a, b in zip(full, again):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("shape", [(3, 6, 200), (4, 9, 33), (2, 5, 129)], ids=lambda s: f"qc{s[0]}x{s[1]}Z{s[2]}")
def test_qc_group_layouts(shape):
    """QC codes with Z > 128 (one thread group per batch) and Z not a multiple of 32."""
    mb, nb, Z = shape
    w = np.array(([3, 2] * nb)[:nb], np.int32)
    w = np.minimum(w, mb)
    code = g.qc(mb, nb, Z, w, seed=Z)
    s2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    for F in (3, 64):
        llr = g.llr(9 + F, 0, F, code.n_vars, s2, g.LLR_I16, 3, 511)
        for es in (0, 1):
            params = P.make_params(8, es, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
            assert_int_parity(code, llr, params, 8, es, 1, 511)


def test_wide_rows_f32_and_unsupported_int():
    """Row degree 12: fp32 path (<= 16) decodes within tolerance; integer paths report UNSUPPORTED."""
    code = g.regular(120, 6, 12, seed=2, remove_4cycles=False)
    s2 = g.ebn0_to_sigma2(3.0, code.rate)
    llr = g.llr(4, 0, 20, code.n_vars, s2, g.LLR_F32)
    params = P.make_params(8, 1, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT)
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr, "compact", "f32", 8, 1, alpha=0.75, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)
    dec = decoder(code)
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(4, P.make_params(8, 0, P.LDPC_MINSUM_OFFSET, 1, 0, 1.0, 63, P.LDPC_LLR_I16))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED


def test_clamp_and_offset_variants_int():
    """Other clamps / offsets than the configs' (Q = 63, 255; beta = 0, 3) on the cfg1 code."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 40)
    for Q, beta in ((63, 0), (255, 3), (511, 0)):
        z = np.clip(llr, -Q, Q)
        params = P.make_params(12, 1, P.LDPC_MINSUM_OFFSET, beta, 0.0, 1.0, Q, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
        assert_int_parity(code, z, params, 12, 1, beta, Q)


def test_qc_odd_batch_and_mixed_convergence():
    """QC resident kernel: odd frame count (a half-empty last pair) on cfg2/cfg3, and a
    2.25 dB batch where frames stop at different iterations."""
    for idx in (2, 3):
        cfg = g.CONFIGS[idx]
        code = cfg.code()
        llr = cfg.llrs(code, 0, 301)
        assert_int_parity(code, llr, _cfg_params(cfg), cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)
    s2 = g.ebn0_to_sigma2(2.25, g.CONFIGS[2].code().rate)
    llr = g.llr(99, 0, 200, g.CONFIGS[2].code().n_vars, s2, g.LLR_I16, 3, 511)
    assert_int_parity(g.CONFIGS[2].code(), llr, _cfg_params(g.CONFIGS[2]), 15, 1, 1, 511)


@pytest.mark.parametrize("fixed", [0, -1], ids=["fixed-bases", "register-bases"])
@pytest.mark.parametrize("fmt", ["compact", "1bit"])
def test_qc_early_stop_buffer_bases(fixed, fmt):
    """The QC early-stop resident kernel with the posterior buffers at a fixed distance and the
    shift table in shared memory (immediate-offset addressing, the default when the code fits)
    and with the buffer bases in registers (tuning.resident_fixed_bases = -1): both bit-exact
    with the oracle on an odd batch whose frames stop at spread-out iterations."""
    code = g.CONFIGS[2].code()
    s2 = g.ebn0_to_sigma2(2.25, code.rate)
    if fmt == "compact":
        llr = g.llr(123, 0, 301, code.n_vars, s2, g.LLR_I16, 3, 511)
        params = P.make_params(15, 1, P.LDPC_MINSUM_OFFSET, 1, llr_type=P.LDPC_LLR_I16)
        Q = 511
    else:
        llr = g.llr(124, 0, 301, code.n_vars, s2, g.LLR_I8, 2, 127)
        params = P.make_params(15, 1, P.LDPC_MINSUM_OFFSET, 1, llr_type=P.LDPC_LLR_I8, msg_format=P.LDPC_MSG_1BIT)
        Q = 127
    ref = assert_int_parity(code, llr, tuned(params, resident_fixed_bases=fixed), 15, 1, 1, Q)
    assert len(np.unique(ref.iters)) >= 4


@pytest.mark.parametrize("fixed", [0, -1], ids=["fixed-bases", "register-bases"])
@pytest.mark.parametrize("fmt", ["compact", "1bit"])
@pytest.mark.parametrize("code_id", ["reg1008", "dvbs2_600"])
def test_general_code_early_stop_buffer_bases(fixed, fmt, code_id):
    """General (CSR) codes with early stop on the barrier-free kernel: column table in shared
    memory with the fixed buffer bases (default) or the register bases, bit-exact with the
    oracle; a row-regular code (one degree dispatch per iteration) and an irregular one."""
    code = g.CONFIGS[1].code() if code_id == "reg1008" else g.dvbs2like(600, 300, 120, 8, 3, seed=6)
    s2 = g.ebn0_to_sigma2(2.5, code.rate)
    if fmt == "compact":
        llr = g.llr(126, 0, 257, code.n_vars, s2, g.LLR_I16, 3, 511)
        params = P.make_params(20, 1, P.LDPC_MINSUM_OFFSET, 1, llr_type=P.LDPC_LLR_I16)
        Q = 511
    else:
        llr = g.llr(127, 0, 257, code.n_vars, s2, g.LLR_I8, 2, 127)
        params = P.make_params(20, 1, P.LDPC_MINSUM_OFFSET, 1, llr_type=P.LDPC_LLR_I8, msg_format=P.LDPC_MSG_1BIT)
        Q = 127
    ref = assert_int_parity(code, llr, tuned(params, resident_fixed_bases=fixed), 20, 1, 1, Q)
    assert len(np.unique(ref.iters)) >= 3


@pytest.mark.parametrize("mb,nb,Z", [(32, 64, 128), (20, 40, 200), (24, 64, 129)],
                         ids=["N8192-fixed", "N8000-Z200-fixed-one-group", "N8256-registers"])
def test_qc_early_stop_fixed_bases_size_boundary(mb, nb, Z):
    """Largest QC code whose posterior buffer fits below the fixed 32 KB offset (N = 8192: 4N =
    32768, fixed bases) and one just above it (N = 8256: buffer bases in registers), both with
    early stop at spread-out iterations, bit-exact with the oracle."""
    code = g.qc(mb, nb, Z, np.full(nb, 3, np.int32), seed=21)
    s2 = g.ebn0_to_sigma2(2.5, code.rate)
    llr = g.llr(125, 0, 96, code.n_vars, s2, g.LLR_I16, 3, 511)
    params = P.make_params(15, 1, P.LDPC_MINSUM_OFFSET, 1, llr_type=P.LDPC_LLR_I16)
    ref = assert_int_parity(code, llr, params, 15, 1, 1, 511)
    assert len(np.unique(ref.iters)) >= 2


@pytest.mark.parametrize("chunk", [1, 2])
def test_stream_l2_chunks(chunk):
    """Streaming kernels decoding the frame tiles in chunks (tuning.stream_chunk_tiles,
    opt-in): int16 with early stop on a QC code (mixed stopping iterations), 1-bit, and
    fp32 -- several tiles plus a ragged last tile, identical to the oracle."""
    tn = {"path": P.LDPC_PATH_STREAM, "stream_chunk_tiles": chunk}
    code = g.qc(6, 12, 37, np.array([3, 4] * 6, np.int32), seed=8)
    s2 = g.ebn0_to_sigma2(2.5, code.rate)
    llr = g.llr(41, 0, 230, code.n_vars, s2, g.LLR_I16, 3, 511)
    params = P.make_params(12, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 0, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT, tuning=tn)
    assert_int_parity(code, llr, params, 12, 1, 1, 511)
    llr = g.llr(43, 0, 230, code.n_vars, s2, g.LLR_I8, 2, 127)
    params = P.make_params(12, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 127, P.LDPC_LLR_I8, P.LDPC_MSG_1BIT, tuning=tn)
    assert_int_parity(code, llr, params, 12, 0, 1, 127)
    llr = g.llr(42, 0, 100, code.n_vars, s2, g.LLR_F32)
    params = P.make_params(10, 1, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT,
                           tuning=tn)
    post, hb, ok, it = gpu_decode(code, llr, params)
    ref = oracle.decode(code, llr, "compact", "f32", 10, 1, alpha=0.75, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)


@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_batched_resident_kernel(cfg_idx):
    """The conflict-free-batch resident kernel (tuning.path = LDPC_PATH_RESIDENT_BATCHED;
    the default flooding kernel accumulates with shared-memory atomics instead) stays
    bit-exact too."""
    tn = {"path": P.LDPC_PATH_RESIDENT_BATCHED}
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 129)
    assert_int_parity(code, llr, tuned(_cfg_params(cfg), **tn), cfg.max_iter, cfg.early_stop, cfg.offset_raw,
                      cfg.clamp)
    for c in small_codes()[:4]:
        z = g.llr(11, 0, 33, c.n_vars, g.ebn0_to_sigma2(1.5, max(c.rate, 0.3)), g.LLR_I16, 3, 511)
        params = P.make_params(10, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT,
                               tuning=tn)
        assert_int_parity(c, z, params, 10, 1, 1, 511)


def test_resident_size_boundary():
    """Largest codes on either side of the resident kernel's shared-memory limit
    (2 N words + reserve <= 227 KB per CTA): N = 26924 resident, N = 27178 streaming."""
    for nb in (212, 214):
        w = np.array(([1, 2, 2] * nb)[:nb], np.int32)
        code = g.qc(64, nb, 127, w, seed=nb)
        assert int(np.max(np.diff(code.row_ptr))) <= 8
        llr = g.llr(77 + nb, 0, 5, code.n_vars, g.ebn0_to_sigma2(2.0, code.rate), g.LLR_I16, 3, 511)
        for es in (0, 1):
            params = P.make_params(6, es, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
            assert_int_parity(code, llr, params, 6, es, 1, 511)


def test_tmem_capacity_falls_back_to_streaming():
    """N = M = 24000 (4,4)-regular: the posteriors fit in shared memory but 94 rows per
    thread need 564 TMEM columns of compact state (> 512), so the planner streams the
    decode (int16 and fp32) -- the layered schedule on the streaming layered kernel; the
    per-edge form, which needs TMEM, is rejected."""
    code = g.regular(24000, 4, 4, seed=3, remove_4cycles=False)
    s2 = g.ebn0_to_sigma2(4.0, 0.5)
    llr = g.llr(8, 0, 3, code.n_vars, s2, g.LLR_I16, 3, 511)
    params = P.make_params(5, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
    assert_int_parity(code, llr, params, 5, 1, 1, 511)
    assert P.ldpc_last_launch_count() > 1                       # streamed
    z = g.llr(9, 0, 3, code.n_vars, s2, g.LLR_F32)
    pf = P.make_params(5, 0, P.LDPC_MINSUM_NORMALIZED, 0, 0.0, 0.75, 0, P.LDPC_LLR_F32, P.LDPC_MSG_COMPACT)
    post, hb, ok, it = gpu_decode(code, z, pf)
    assert P.ldpc_last_launch_count() > 1
    ref = oracle.decode(code, z, "compact", "f32", 5, 0, alpha=0.75, nthreads=NT)
    assert_f32_exact(post, hb, ok, it, ref)
    dec = decoder(code)
    bad = P.make_params(5, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_FULL)
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(3, bad)
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED
    # the layered schedule falls back to the streaming layered kernel
    lay = P.make_params(5, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT,
                        P.LDPC_SCHED_LAYERED)
    post, hb, ok, it = gpu_decode(code, llr, lay)
    ref = oracle.decode(code, llr.astype(np.int32), "layered", "int", 5, 1, 1, 511, nthreads=NT)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(it, ref.iters)


def test_high_column_degree_batched_kernel():
    """Column degree 20 at Q = 511: 2Q(dv+1) >= 0x4000, so the (unbiased) batched resident
    kernel runs; the streaming integer path rejects it (biased lanes would overflow)."""
    code = g.regular(80, 20, 8, seed=3, remove_4cycles=False)
    llr = g.llr(5, 0, 33, code.n_vars, 0.9, g.LLR_I16, 3, 511)
    params = P.make_params(8, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
    assert_int_parity(code, llr, params, 8, 1, 1, 511)
    # the resident layered kernel keeps unbiased lanes too
    lay = P.make_params(8, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT,
                        P.LDPC_SCHED_LAYERED)
    post, hb, ok, it = gpu_decode(code, llr, lay)
    ref = oracle.decode(code, llr.astype(np.int32), "layered", "int", 8, 1, 1, 511, nthreads=NT)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(it, ref.iters)
    dec = decoder(code)
    with pytest.raises(P.LdpcError) as e:
        dec.workspace(33, tuned(params, path=P.LDPC_PATH_STREAM))
    assert e.value.status == P.LDPC_ERR_UNSUPPORTED


def test_many_iterations():
    """200 iterations (no early stop) on the cfg1 code, resident and streaming."""
    cfg = g.CONFIGS[1]
    code = cfg.code()
    llr = cfg.llrs(code, 0, 40)
    params = P.make_params(200, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, P.LDPC_MSG_COMPACT)
    assert_int_parity(code, llr, params, 200, 0, 1, 511)


def test_concurrent_host_api_calls_on_one_code():
    """Two host threads decode different frame sets through ldpc_decode_batch_host on the
    same code object, each with its own workspace, stream and buffers: both bit-exact."""
    import threading
    cfg = g.CONFIGS[2]
    code = cfg.code()
    dec = decoder(code)
    params = P.params_for_config(cfg)
    results = {}

    def worker(idx):
        llr = cfg.llrs(code, 1000 * idx, 600)
        nb = P.ldpc_decode_host_workspace_size(dec.handle, 600, params)
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
        lh = torch.from_numpy(llr).pin_memory()
        hb = torch.empty((600, dec.wpf), dtype=torch.int32).pin_memory()
        ok = torch.empty(600, dtype=torch.uint8).pin_memory()
        it = torch.empty(600, dtype=torch.int32).pin_memory()
        post = torch.empty((600, code.n_vars), dtype=torch.int16).pin_memory()
        s = torch.cuda.Stream(device="cuda:0")
        for _ in range(3):
            P.ldpc_decode_batch_host(dec.handle, params, 600, lh.data_ptr(), hb.data_ptr(), post.data_ptr(),
                                     ok.data_ptr(), it.data_ptr(), ws.data_ptr(), nb, s.cuda_stream)
        s.synchronize()
        results[idx] = (llr, post.numpy().copy(), hb.numpy().view(np.uint32).copy(), ok.numpy().copy(),
                        it.numpy().copy())

    th = [threading.Thread(target=worker, args=(i,)) for i in (1, 2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for idx in (1, 2):
        llr, post, hb, ok, it = results[idx]
        ref = oracle_decode_int(code, llr, cfg.max_iter, cfg.early_stop, cfg.offset_raw, cfg.clamp)
        np.testing.assert_array_equal(post.astype(np.int32), ref.post)
        np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))
        np.testing.assert_array_equal(ok, ref.ok)
        np.testing.assert_array_equal(it, ref.iters)


def test_plain_c_consumer():
    """examples/decode_c.c: the C ABI used from plain C (no Python, no PyTorch) -- code
    creation from a QC shift table, both decode entry points, error counters."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "decode_c")
    if not os.path.exists(exe):                       # build it (gcc + the in-tree libldpc.so)
        subprocess.check_call(["make", "-C", root, "examples/decode_c"], stdout=subprocess.DEVNULL)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


@pytest.mark.parametrize("kind", ["int16", "int16-full", "1bit-msgs"])
def test_resident_grid_loop(kind):
    """tuning.resident_waves = 1 caps the resident grid at one wave (blocks/SM x SMs), so every
    CTA loops over several frame pairs: outputs (and, for 1bit-msgs, the exported messages) of
    all frames must still match."""
    code = small_codes()[1]                        # regular (3,6), N = 96
    F = 4 * 148 * 32 + 7                           # well above one wave at any occupancy, odd
    s2 = g.ebn0_to_sigma2(2.0, code.rate)
    tn = {"resident_waves": 1}
    if kind == "1bit-msgs":
        llr = g.llr(7, 0, F, code.n_vars, s2, g.LLR_I8, 2, 127)
        params = P.make_params(8, 0, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 127, P.LDPC_LLR_I8, P.LDPC_MSG_1BIT, tuning=tn)
        dec = decoder(code)
        out, msg = dec.decode_messages(torch.from_numpy(llr).cuda(), params)
        torch.cuda.synchronize()
        assert P.ldpc_last_launch_count() == 1
        picks = np.r_[0:3, F - 3:F]
        ref = oracle.decode(code, llr[picks].astype(np.int32), "compact", "int", 8, 0, 1, 127, trace=True, nthreads=NT)
        np.testing.assert_array_equal(msg.cpu().numpy()[picks].astype(np.int32), ref.trace_msg[:, 7, :])
        np.testing.assert_array_equal(out.posteriors.cpu().numpy()[picks].astype(np.int32), ref.post)
        return
    llr = g.llr(6, 0, F, code.n_vars, s2, g.LLR_I16, 3, 511)
    fmt = P.LDPC_MSG_FULL if kind == "int16-full" else P.LDPC_MSG_COMPACT
    params = P.make_params(8, 1, P.LDPC_MINSUM_OFFSET, 1, 0.0, 1.0, 511, P.LDPC_LLR_I16, fmt, tuning=tn)
    post, hb, ok, it = gpu_decode(code, llr, params)
    assert P.ldpc_last_launch_count() == 1
    ref = oracle.decode(code, llr.astype(np.int32), "compact", "int", 8, 1, 1, 511, nthreads=NT)
    np.testing.assert_array_equal(it, ref.iters)
    np.testing.assert_array_equal(ok, ref.ok)
    np.testing.assert_array_equal(post.astype(np.int32), ref.post)
    np.testing.assert_array_equal(hb, oracle.pack_bits(ref.bits))


@pytest.mark.parametrize("cfg_idx", [1, 2, 4, 5])
def test_decode_inside_cuda_graph(cfg_idx):
    """ldpc_decode_batch is stream-ordered and allocation-free, so it can be captured in a CUDA
    graph (the bench times cfg1 that way): two batches captured back to back -- resident,
    streaming with programmatic dependent launches (cfg4) and fp32 (cfg5) -- replayed, and
    their outputs equal to direct decodes."""
    cfg = g.CONFIGS[cfg_idx]
    code = cfg.code()
    F = {1: 300, 2: 200, 4: 70, 5: 40}[cfg_idx]
    params = _cfg_params(cfg)
    if cfg_idx >= 4:
        params.max_iter = 12
    dec = P.Decoder(code, 0)
    llrs = [torch.from_numpy(cfg.llrs(code, 5000 * (b + 1), F)).cuda() for b in range(2)]
    ref = []
    for x in llrs:
        o = dec.decode(x, params)
        torch.cuda.synchronize()
        ref.append((o.posteriors.clone(), o.hard_bits.clone(), o.syndrome_ok.clone(), o.iterations.clone()))
    outs = [dec.alloc_outputs(F, params.llr_type, posteriors=True) for _ in range(2)]
    dec2 = P.Decoder(code, 0)              # its own workspace per batch: both decodes in one graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dec.decode(llrs[0], params, outs[0])
        dec2.decode(llrs[1], params, outs[1])
    torch.cuda.synchronize()
    for o in outs:
        o.posteriors.zero_()
        o.hard_bits.zero_()
        o.iterations.fill_(-1)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        dec.decode(llrs[0], params, outs[0])
        dec2.decode(llrs[1], params, outs[1])
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    for o, (rp, rh, rk, ri) in zip(outs, ref):
        assert torch.equal(o.posteriors, rp)
        assert torch.equal(o.hard_bits, rh)
        assert torch.equal(o.syndrome_ok, rk)
        assert torch.equal(o.iterations, ri)
    dec2.close()
    dec.close()

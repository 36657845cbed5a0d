"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every pin is independent of the oracle's own code: hand-evaluated rows and
trajectories (tests/golden/, each cited), Eq.(1) evaluated literally vs the
two-minima/compact form, the paper's stated equivalences, exact
max-marginals on tree Tanner graphs, a closed-form noiseless trajectory,
stopping rules, and exhaustive ML decoding of a tiny code.
"""
import itertools
import json
import os

import numpy as np
import pytest

import ldpcgen as g
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------- check-row pins
@pytest.mark.parametrize("row", _load("check_rows.json")["rows"], ids=lambda r: r["cite"][:40])
def test_check_rows_golden(row):
    mode = row["mode"]
    kw = dict(mode=mode, beta=row["beta"], clamp=row["clamp"], alpha=row.get("alpha", 1.0))
    naive = oracle.check_naive(row["q"], **kw)
    L, A, B, idx, s = oracle.check_compact(row["q"], **kw)
    np.testing.assert_allclose(naive, row["L"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(L, row["L"], rtol=0, atol=1e-12)
    assert A == pytest.approx(row["A"]) and B == pytest.approx(row["B"])
    if row["idx"] is not None and row["A"] != row["B"]:
        assert idx == row["idx"]


def _random_rows(rng, n, mode):
    for _ in range(n):
        dc = int(rng.integers(2, 10))
        if mode == "int":
            q = rng.integers(-40, 41, dc)
            if rng.random() < 0.3:      # force ties and zeros
                q[rng.integers(0, dc)] = q[rng.integers(0, dc)]
            if rng.random() < 0.1:
                q[rng.integers(0, dc)] = 0
        else:
            q = rng.normal(0, 5, dc)
            if rng.random() < 0.2:
                q[rng.integers(0, dc)] = -q[rng.integers(0, dc)]
        yield q


@pytest.mark.parametrize("mode", ["int", "f64", "f32"])
def test_naive_eq1_equals_compact_form(mode):
    """SPEC S:294 / SURVEY §8(c): Eq.(1) evaluated literally (O(dc^2)) equals the
    §5 compact form (two minima, argmin, signs) on >= 2e4 random rows."""
    rng = np.random.default_rng(7)
    mism = 0
    for q in _random_rows(rng, 20000, mode):
        for beta, clamp, alpha in ([(0, 0, 1.0), (1, 0, 1.0), (2, 31, 1.0)] if mode == "int"
                                   else [(0, 0, 1.0), (0, 0, 0.75), (0.5, 0, 0.8)]):
            a = oracle.check_naive(q, mode, beta, clamp, alpha)
            b = oracle.check_compact(q, mode, beta, clamp, alpha)[0]
            mism += int(not np.array_equal(a, b))
    assert mism == 0


def test_compact_structure_property():
    """P:259-260 'all have the same absolute value except one':
    at most two distinct |L| per check, the larger exactly at ñ when min1 < min2, A <= B."""
    rng = np.random.default_rng(11)
    for q in _random_rows(rng, 10000, "int"):
        L, A, B, idx, s = oracle.check_compact(q, "int", beta=1, clamp=63)
        mags = np.abs(L)
        assert len(set(mags.tolist())) <= 2
        assert A <= B
        srt = np.sort(np.abs(q))
        if srt[0] < srt[1] and A < B:
            assert mags[idx] == B and np.all(np.delete(mags, idx) == A)
            assert idx == int(np.argmin(np.abs(q)))
        # signs: s_mn = prod_{n' != n} sgn(q_n') with sgn(0)=+1
        sg = np.where(q < 0, -1, 1)
        assert np.array_equal(s, np.prod(sg) * sg)


# ------------------------------------------------------ toy trajectories
ENGINES = ["twoscan_naive", "twoscan", "singlescan", "compact"]


@pytest.mark.parametrize("case", _load("toy_trajectories.json")["cases"], ids=lambda c: c["cite"])
@pytest.mark.parametrize("engine", ENGINES)
def test_toy_trajectories(case, engine):
    code = g.from_dense(_load("toy_trajectories.json")["code"])
    r = oracle.decode(code, np.array([case["z0"]]), engine=engine, mode=case["mode"], max_iter=2,
                      beta=case["beta"], trace=True)
    np.testing.assert_allclose(r.trace_post[0], case["post"], rtol=0, atol=1e-12)


def test_hard_decision_and_syndrome_examples():
    gd = _load("decode_core.json")
    # hard decision: a 1-variable "code" is not allowed (dc>=2), so use the toy code with
    # max_iter-free inspection: early_stop at k=0 outputs x̂(Z0) (D10).
    code = g.from_dense([[1, 1, 0], [0, 1, 1]])
    z = np.array([gd["hard_decision"]["z"]])
    r = oracle.decode(code, z, engine="compact", mode="f64", max_iter=1, early_stop=1)
    # x̂ = [0,1,1]: row0 0^1 = 1 -> not a codeword, so one iteration runs; check the
    # k=0 decision through a zero-iteration-equivalent: decode with alpha=0 keeps L=Z0.
    r0 = oracle.decode(code, z, engine="compact", mode="f64", max_iter=1, alpha=0.0)
    assert r0.bits[0].tolist() == gd["hard_decision"]["bits"]
    assert r.iters[0] >= 1
    # syndrome: x=[1,1,0] gives s=[0,1] -> not a codeword; x=[1,1,1] is a codeword
    sy = gd["syndrome"]
    z_from_x = np.where(np.array(sy["x"]) == 1, -1.0, 1.0)[None]
    r1 = oracle.decode(g.from_dense(sy["H"]), z_from_x, engine="compact", mode="f64", max_iter=1, early_stop=1,
                       alpha=0.0)
    assert int(r1.ok[0]) == int(not any(sy["s"]))
    r2 = oracle.decode(g.from_dense(sy["H"]), -np.ones((1, 3)), engine="compact", mode="f64", max_iter=1,
                       early_stop=1)
    assert r2.ok[0] == 1 and r2.iters[0] == 0


# ------------------------------------------ engine equivalence
def _codes_small():
    return [
        g.from_dense([[1, 1, 0], [0, 1, 1]], name="toy"),
        g.regular(96, 3, 6, seed=5),
        g.regular(48, 3, 6, seed=9, remove_4cycles=False),
        g.qc(4, 8, 7, np.array([2, 3, 2, 3, 2, 2, 3, 2], np.int32), seed=3),
        g.dvbs2like(64, 32, 16, 5, 3, seed=4),
    ]


@pytest.mark.parametrize("code", _codes_small(), ids=lambda c: c.name)
@pytest.mark.parametrize("beta,clamp", [(0, 511), (1, 31), (2, 15)])
def test_int_engines_bit_identical(code, beta, clamp):
    """PAPER.md P:338 'fully equivalent to the original min-sum algorithm':
    two-scan (naive Eq.(1)), two-scan (two minima), single-scan and compact
    single-scan give bit-identical per-iteration posteriors and messages,
    hard bits, syndrome flags and iteration counts in fixed point."""
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    z0 = g.llr(77, 0, 30, code.n_vars, sigma2, g.LLR_I16, 3, 511).astype(np.int32)
    ref = oracle.decode(code, z0, "twoscan_naive", "int", 30, 0, beta, clamp, trace=True)
    for eng in ENGINES[1:]:
        r = oracle.decode(code, z0, eng, "int", 30, 0, beta, clamp, trace=True)
        assert np.array_equal(r.trace_post, ref.trace_post), eng
        assert np.array_equal(r.trace_msg, ref.trace_msg), eng
        assert np.array_equal(r.bits, ref.bits) and np.array_equal(r.ok, ref.ok)
        assert np.array_equal(r.iters, ref.iters)
    # with early stop too
    ref = oracle.decode(code, z0, "twoscan_naive", "int", 30, 1, beta, clamp)
    r = oracle.decode(code, z0, "compact", "int", 30, 1, beta, clamp)
    for a, b in [(r.post, ref.post), (r.bits, ref.bits), (r.ok, ref.ok), (r.iters, ref.iters)]:
        assert np.array_equal(a, b)


def test_trace_messages_have_compact_structure():
    """Every check's messages in a real decode trace take <= 2 magnitudes."""
    code = g.regular(96, 3, 6, seed=5)
    z0 = g.llr(3, 0, 5, code.n_vars, 0.8, g.LLR_I16, 3, 511).astype(np.int32)
    r = oracle.decode(code, z0, "compact", "int", 10, 0, 1, 511, trace=True)
    for f in range(5):
        for k in range(10):
            for m in range(code.n_checks):
                row = np.abs(r.trace_msg[f, k, code.row_ptr[m]:code.row_ptr[m + 1]])
                assert len(np.unique(row)) <= 2


@pytest.mark.parametrize("code", _codes_small()[1:3], ids=lambda c: c.name)
def test_float_engines(code):
    """compact == single-scan exactly in float (same arithmetic);
    single-scan vs two-scan within 1e-9 relative in float64."""
    sigma2 = g.ebn0_to_sigma2(1.5, code.rate)
    z0 = g.llr(8, 0, 20, code.n_vars, sigma2, g.LLR_F64)
    for alpha in (1.0, 0.8, 0.75):
        ts = oracle.decode(code, z0, "twoscan", "f64", 30, 0, alpha=alpha, trace=True)
        ss = oracle.decode(code, z0, "singlescan", "f64", 30, 0, alpha=alpha, trace=True)
        cp = oracle.decode(code, z0, "compact", "f64", 30, 0, alpha=alpha, trace=True)
        assert np.array_equal(ss.trace_post, cp.trace_post)
        assert np.array_equal(ss.trace_msg, cp.trace_msg)
        scale = 1.0 + np.abs(ts.trace_post)
        assert np.max(np.abs(ss.trace_post - ts.trace_post) / scale) < 1e-9


def test_f32_mode_tracks_f64():
    """Reading D11: the fp32 oracle (one RN rounding per op) stays within the
    north-star tolerance |dL| <= 1e-4 (1+|L|) of the float64 oracle on a
    cfg5-shaped workload (same code family, alpha = 0.75, 50 iterations)."""
    code = g.dvbs2like(2400, 1200, 480, 8, 3, seed=1)
    z0 = g.llr(2005, 0, 6, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_F32)
    a = oracle.decode(code, z0.astype(np.float64), "compact", "f64", 50, 0, alpha=0.75)
    b = oracle.decode(code, z0, "compact", "f32", 50, 0, alpha=0.75)
    assert np.max(np.abs(a.post - b.post) / (1 + np.abs(a.post))) < 1e-4


# ---------------------------------------- exact results (tree codes, ML)
def _random_tree_code(rng, n_checks=4):
    """Random tree-structured Tanner graph: each new check touches exactly one
    existing variable plus fresh ones, so the graph has no cycles."""
    rows = [[0, 1, 2]]
    nv = 3
    for _ in range(n_checks - 1):
        anchor = int(rng.integers(0, nv))
        k = int(rng.integers(1, 3))
        rows.append([anchor] + list(range(nv, nv + k)))
        nv += k
    H = np.zeros((len(rows), nv), np.uint8)
    for m, r in enumerate(rows):
        H[m, r] = 1
    return g.from_dense(H, name="tree")


def _codewords(H):
    M, N = H.shape
    words = np.array(list(itertools.product([0, 1], repeat=N)), np.uint8)
    return words[((words @ H.T) % 2 == 0).all(axis=1)]


def test_tree_posteriors_are_exact_max_marginals():
    """On a cycle-free Tanner graph, plain min-sum (beta=0, no clamp) computes exact
    max-marginals once the iteration count exceeds the tree depth:
    Z_n = max_{c in C, c_n=0} m(c) - max_{c in C, c_n=1} m(c),  m(c) = 1/2 sum (1-2c_i) Z0_i.
    Brute force over all codewords; exact in integer arithmetic."""
    rng = np.random.default_rng(123)
    for t in range(500):
        code = _random_tree_code(rng, n_checks=int(rng.integers(2, 6)))
        H = code.dense()
        C = _codewords(H)
        z0 = rng.integers(-20, 21, (1, code.n_vars))
        r = oracle.decode(code, z0, "compact", "int", 12, 0, 0, 0)
        mc = ((1 - 2 * C.astype(np.int64)) * z0).sum(axis=1)   # = 2 m(c)
        want = np.array([(mc[C[:, n] == 0].max() - mc[C[:, n] == 1].max()) // 2 for n in range(code.n_vars)])
        assert np.array_equal(r.post[0], want), t


def test_noiseless_closed_form_on_cfg1_code():
    """Constant input c on a (dv,dc)-regular code: every message equals r_k with
    r_1 = clamp(c - beta), r_{k+1} = clamp(c + (dv-1) r_k - beta), L_k = c + dv r_k."""
    gd = _load("decode_core.json")["noiseless_closed_form"]
    code = g.CONFIGS[1].code()
    K = len(gd["L"])
    z0 = np.full((1, code.n_vars), gd["c"], np.int32)
    r = oracle.decode(code, z0, "compact", "int", K, 0, gd["beta"], gd["Q"], trace=True)
    for k in range(K):
        assert np.all(r.trace_post[0, k] == gd["L"][k])
    # and the recurrence itself reproduces the fixture
    rk, Ls = min(max(gd["c"] - gd["beta"], 0), gd["Q"]), []
    for k in range(K):
        Ls.append(gd["c"] + gd["dv"] * rk)
        rk = min(max(gd["c"] + (gd["dv"] - 1) * rk - gd["beta"], 0), gd["Q"])
    assert Ls == gd["L"]


def test_stopping_rules():
    """SPEC S:234-235, S:480 (reading D10): noiseless frames stop at k=0 with a zero
    syndrome; capped runs report max_iter; with early_stop=0 every frame runs max_iter."""
    code = g.regular(96, 3, 6, seed=5)
    z0 = np.full((3, 96), 5, np.int32)
    for eng in ENGINES:
        r = oracle.decode(code, z0, eng, "int", 10, 1, 1, 511)
        assert np.all(r.iters == 0) and np.all(r.ok == 1) and np.all(r.bits == 0)
        r = oracle.decode(code, z0, eng, "int", 10, 0, 1, 511)
        assert np.all(r.iters == 10) and np.all(r.ok == 1)
    # strongly contradictory input: all bits flipped on an odd-weight row set can't be fixed in 1 iteration
    bad = np.full((1, 96), 5, np.int32)
    bad[0, code.col_idx[code.row_ptr[0]]] = -200
    r = oracle.decode(code, bad, "compact", "int", 1, 1, 0, 0)
    assert r.iters[0] == 1 and r.ok[0] == 0


def _gf2_nullspace(H):
    H = H.copy() % 2
    M, N = H.shape
    pivots = []
    r = 0
    for c in range(N):
        p = next((i for i in range(r, M) if H[i, c]), None)
        if p is None:
            continue
        H[[r, p]] = H[[p, r]]
        for i in range(M):
            if i != r and H[i, c]:
                H[i] ^= H[r]
        pivots.append(c)
        r += 1
        if r == M:
            break
    free = [c for c in range(N) if c not in pivots]
    basis = []
    for fcol in free:
        v = np.zeros(N, np.uint8)
        v[fcol] = 1
        for i, pc in enumerate(pivots):
            v[pc] = H[i, fcol]
        basis.append(v)
    return np.array(basis, np.uint8)


def test_exhaustive_ml_tiny_code_high_snr():
    """North star: 'exhaustive ML decoding of a tiny code at high SNR'.  On a
    (3,6)-regular N=24 code at 5 dB, compact single-scan offset min-sum agrees with
    the exact ML codeword (argmax_c sum (1-2c) Z0) on >= 98% of frames, and every
    frame it declares converged is a codeword."""
    code = g.regular(24, 3, 6, seed=21, remove_4cycles=False)
    H = code.dense()
    B = _gf2_nullspace(H)
    assert ((B @ H.T) % 2 == 0).all()
    k = B.shape[0]
    coeffs = np.array(list(itertools.product([0, 1], repeat=k)), np.uint8)
    C = (coeffs @ B) % 2
    F = 2000
    z = g.llr(31, 0, F, 24, g.ebn0_to_sigma2(5.0, 0.5), g.LLR_F64)
    ml = C[np.argmax((1 - 2 * C.astype(np.float64)) @ z.T, axis=0)]
    zi = np.clip(np.rint(z * 8), -511, 511).astype(np.int32)
    r = oracle.decode(code, zi, "compact", "int", 30, 1, 1, 511)
    agree = np.mean(np.all(r.bits == ml, axis=1))
    assert agree >= 0.98, agree
    conv = r.ok == 1
    assert np.all(((r.bits[conv].astype(np.int64) @ H.T) % 2) == 0)


# ------------------------------------------------- layered schedule (§8(f2))
@pytest.mark.parametrize("case", _load("layered_toy.json")["cases"], ids=lambda c: c["cite"])
@pytest.mark.parametrize("engine", ["layered_full", "layered"])
def test_layered_toy_trajectories(case, engine):
    """Hand-evaluated in-place trajectories (tests/golden/layered_toy.json, reading D25)."""
    code = g.from_dense(_load("layered_toy.json")["code"])
    r = oracle.decode(code, np.array([case["z0"]]), engine=engine, mode=case["mode"], max_iter=2,
                      beta=case["beta"], trace=True)
    np.testing.assert_allclose(r.trace_post[0], case["post"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("code", _codes_small(), ids=lambda c: c.name)
@pytest.mark.parametrize("beta,clamp", [(0, 511), (1, 31)])
def test_layered_compact_equals_full_messages(code, beta, clamp):
    """The compact state recovers every previous message exactly, so the
    layered schedule over the compact state is bit-identical to layered with stored
    per-edge L_mn and the literal Eq.(1) rule, per iteration, with and without early stop."""
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    z0 = g.llr(78, 0, 30, code.n_vars, sigma2, g.LLR_I16, 3, 511).astype(np.int32)
    for es in (0, 1):
        a = oracle.decode(code, z0, "layered_full", "int", 20, es, beta, clamp, trace=True)
        b = oracle.decode(code, z0, "layered", "int", 20, es, beta, clamp, trace=True)
        for x, y in [(a.trace_post, b.trace_post), (a.trace_msg, b.trace_msg), (a.post, b.post), (a.bits, b.bits),
                     (a.ok, b.ok), (a.iters, b.iters)]:
            assert np.array_equal(x, y)


def test_layered_equals_flooding_when_rows_share_no_variable():
    """With every column in one row there is nothing for a later row to see: the
    layered and flooding schedules coincide exactly."""
    rng = np.random.default_rng(7)
    perm = rng.permutation(60)
    H = np.zeros((12, 60), np.uint8)
    for m in range(12):
        H[m, perm[5 * m:5 * m + 5]] = 1
    code = g.from_dense(H, name="disjoint")
    z0 = rng.integers(-60, 61, (20, 60)).astype(np.int32)
    a = oracle.decode(code, z0, "layered", "int", 6, 0, 1, 127, trace=True)
    b = oracle.decode(code, z0, "compact", "int", 6, 0, 1, 127, trace=True)
    assert np.array_equal(a.trace_post, b.trace_post)


def test_layered_tree_posteriors_are_exact_max_marginals():
    """On a cycle-free Tanner graph the layered schedule, like flooding, reaches the
    exact max-marginals (plain min-sum) once enough iterations have run."""
    rng = np.random.default_rng(321)
    for t in range(300):
        code = _random_tree_code(rng, n_checks=int(rng.integers(2, 6)))
        C = _codewords(code.dense())
        z0 = rng.integers(-20, 21, (1, code.n_vars))
        r = oracle.decode(code, z0, "layered", "int", 12, 0, 0, 0)
        mc = ((1 - 2 * C.astype(np.int64)) * z0).sum(axis=1)
        want = np.array([(mc[C[:, n] == 0].max() - mc[C[:, n] == 1].max()) // 2 for n in range(code.n_vars)])
        assert np.array_equal(r.post[0], want), t


def test_layered_row_order_matters_and_stopping():
    """Layered is NOT the flooding schedule on a loopy code -- it differs after
    the first row that sees an earlier update -- yet noiseless frames still stop at k=0
    and converged hard decisions agree with flooding at high SNR."""
    code = g.regular(96, 3, 6, seed=5)
    z0 = g.llr(5, 0, 8, code.n_vars, g.ebn0_to_sigma2(1.5, code.rate), g.LLR_I16, 3, 511).astype(np.int32)
    a = oracle.decode(code, z0, "layered", "int", 3, 0, 1, 511)
    b = oracle.decode(code, z0, "compact", "int", 3, 0, 1, 511)
    assert not np.array_equal(a.post, b.post)
    r = oracle.decode(code, np.full((3, code.n_vars), 12, np.int32), "layered", "int", 10, 1, 1, 511)
    assert np.all(r.iters == 0) and np.all(r.ok == 1)
    z0 = g.llr(6, 0, 40, code.n_vars, g.ebn0_to_sigma2(5.0, code.rate), g.LLR_I16, 3, 511).astype(np.int32)
    a = oracle.decode(code, z0, "layered", "int", 30, 1, 1, 511)
    b = oracle.decode(code, z0, "compact", "int", 30, 1, 1, 511)
    both = (a.ok == 1) & (b.ok == 1)
    assert both.sum() >= 38 and np.array_equal(a.bits[both], b.bits[both])
    assert a.iters[both].mean() <= b.iters[both].mean()


# ------------------------- per-iteration schedules, integer normalization (§8(f3))
@pytest.mark.parametrize("case", _load("schedules_toy.json")["cases"], ids=lambda c: c["cite"])
@pytest.mark.parametrize("engine", ENGINES)
def test_schedule_toy_trajectories(case, engine):
    """Hand-evaluated trajectories with beta_k / lambda_k schedules and floor(lambda |L|)
    (tests/golden/schedules_toy.json, reading D27)."""
    gd = _load("schedules_toy.json")
    code = g.from_dense(gd["code"])
    r = oracle.decode(code, np.array([gd["z0"]]), engine=engine, mode="int", max_iter=2, trace=True,
                      beta_sched=case["beta_sched"], alpha_sched=case["alpha_sched"])
    np.testing.assert_array_equal(r.trace_post[0], case["post"])


def test_int_normalized_check_row():
    """floor(3/4 * min) on a hand-evaluated 3-edge row: q = [7, -3, 9] -> [-2, 5, -2]."""
    out = oracle.check_naive(np.array([7, -3, 9]), "int", alpha=0.75)
    assert out.tolist() == [-2, 5, -2]
    msgs, A, B, idx, s = oracle.check_compact(np.array([7, -3, 9]), "int", alpha=0.75)
    assert msgs.tolist() == [-2, 5, -2] and (A, B, idx) == (2, 5, 1)


@pytest.mark.parametrize("code", _codes_small()[:3], ids=lambda c: c.name)
def test_schedules_engines_bit_identical(code):
    """P:338 equivalence holds iteration by iteration under beta_k / lambda_k schedules
    (integer, dyadic lambda): naive two-scan == compact single-scan, and layered full-L ==
    layered compact; a constant schedule equals the scalar parameters."""
    sigma2 = g.ebn0_to_sigma2(1.5, max(code.rate, 0.3))
    z0 = g.llr(79, 0, 20, code.n_vars, sigma2, g.LLR_I16, 3, 511).astype(np.int32)
    K = 12
    bs = [2, 2, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0]
    al = [0.5, 0.625, 0.75, 0.75, 0.875, 0.875, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0]
    a = oracle.decode(code, z0, "twoscan_naive", "int", K, 0, 0, 511, trace=True, beta_sched=bs, alpha_sched=al)
    b = oracle.decode(code, z0, "compact", "int", K, 0, 0, 511, trace=True, beta_sched=bs, alpha_sched=al)
    assert np.array_equal(a.trace_post, b.trace_post) and np.array_equal(a.trace_msg, b.trace_msg)
    a = oracle.decode(code, z0, "layered_full", "int", K, 1, 0, 511, trace=True, beta_sched=bs, alpha_sched=al)
    b = oracle.decode(code, z0, "layered", "int", K, 1, 0, 511, trace=True, beta_sched=bs, alpha_sched=al)
    assert np.array_equal(a.trace_post, b.trace_post) and np.array_equal(a.iters, b.iters)
    c1 = oracle.decode(code, z0, "compact", "int", K, 0, 1, 511, alpha=0.75, trace=True)
    c2 = oracle.decode(code, z0, "compact", "int", K, 0, 0, 511, trace=True, beta_sched=[1] * K, alpha_sched=[0.75] * K)
    assert np.array_equal(c1.trace_post, c2.trace_post)


def test_float_schedule_matches_scalar_and_twoscan():
    code = g.regular(96, 3, 6, seed=5)
    z0 = g.llr(8, 0, 10, code.n_vars, g.ebn0_to_sigma2(1.5, code.rate), g.LLR_F64)
    al = np.linspace(0.6, 0.9, 15)
    ts = oracle.decode(code, z0, "twoscan", "f64", 15, 0, trace=True, alpha_sched=al)
    cp = oracle.decode(code, z0, "compact", "f64", 15, 0, trace=True, alpha_sched=al)
    assert np.max(np.abs(ts.trace_post - cp.trace_post) / (1 + np.abs(ts.trace_post))) < 1e-9
    s1 = oracle.decode(code, z0, "compact", "f64", 15, 0, alpha=0.8, trace=True)
    s2 = oracle.decode(code, z0, "compact", "f64", 15, 0, trace=True, alpha_sched=[0.8] * 15)
    assert np.array_equal(s1.trace_post, s2.trace_post)


# ---------------------------------------- reading D28: fp32 posterior sums
def _rn_f32(q):
    """Round a Fraction to the nearest float32, ties to even (no double rounding)."""
    from fractions import Fraction
    a = np.float32(float(q))
    best = None
    for c in (np.nextafter(a, np.float32(-np.inf)), a, np.nextafter(a, np.float32(np.inf))):
        d = abs(Fraction(float(c)) - q)
        key = (d, int(np.array(c, np.float32).view(np.uint32)) & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return np.float32(best[1])


def test_f32_posterior_sum_is_exact_then_rounded_once():
    """D28: Z_n = Z0_n + sum_m L_mn is the exact rational sum rounded once to fp32 (pinned
    against Fraction arithmetic, not against the oracle's own grid), for terms with
    2^-11 <= |x| <= 2^20 where the 2^-34 grid holds every fp32 value exactly; the result does
    not depend on the order of the terms; magnitudes beyond 2^20 saturate."""
    from fractions import Fraction
    rng = np.random.default_rng(28)
    for trial in range(400):
        n = int(rng.integers(1, 12))
        mag = np.exp2(rng.uniform(-11, 20, n)).astype(np.float32)
        x = (mag * rng.choice([-1, 1], n)).astype(np.float32)
        x = np.clip(x, -2.0 ** 20, 2.0 ** 20).astype(np.float32)
        exact = sum((Fraction(float(v)) for v in x), Fraction(0))
        want = _rn_f32(exact)
        got = oracle.f32_exact_sum(x)
        assert got.view(np.uint32) == want.view(np.uint32), (x, got, want)
        perm = x[rng.permutation(n)]
        assert oracle.f32_exact_sum(perm).view(np.uint32) == got.view(np.uint32)
    # a sequential fp32 sum is order-dependent where the exact sum is not
    x = np.array([1.0, 2.0 ** -24, 2.0 ** -24], np.float32)
    assert oracle.f32_exact_sum(x) == np.float32(1.0 + 2.0 ** -23)
    assert np.float32(np.float32(1.0) + np.float32(2.0 ** -24)) + np.float32(2.0 ** -24) == np.float32(1.0)
    # saturation at 2^20 and terms far below the grid
    assert oracle.f32_exact_sum(np.array([3e7], np.float32)) == np.float32(2.0 ** 20)
    assert oracle.f32_exact_sum(np.array([2.5, 1e-12], np.float32)) == np.float32(2.5)


def test_f32_flooding_engines_order_free():
    """D28 consequences in fp32: the compact single-scan equals the per-edge single-scan bit
    for bit (same messages, exact sums), and since the order of the rows does not enter an
    exact sum, permuting the rows of H leaves every posterior unchanged (a sequential fp32
    sum would not be order-free)."""
    code = g.dvbs2like(600, 300, 120, 8, 3, seed=6)
    z0 = g.llr(2005, 0, 8, code.n_vars, g.ebn0_to_sigma2(1.0, code.rate), g.LLR_F32)
    a = oracle.decode(code, z0, "compact", "f32", 20, 0, alpha=0.75)
    b = oracle.decode(code, z0, "singlescan", "f32", 20, 0, alpha=0.75)
    assert np.array_equal(a.post.view(np.uint32), b.post.view(np.uint32))
    rng = np.random.default_rng(3)
    order = rng.permutation(code.n_checks)
    rows = [code.col_idx[code.row_ptr[m]:code.row_ptr[m + 1]] for m in order]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    perm = g.Code(code.n_vars, code.n_checks, rp, np.concatenate(rows).astype(np.int32), name="perm")
    c = oracle.decode(perm, z0, "compact", "f32", 20, 0, alpha=0.75)
    assert np.array_equal(a.post.view(np.uint32), c.post.view(np.uint32))

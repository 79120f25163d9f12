"""GPU parity: every CUDA stage against the oracle (the C restatement pinned
to the reference in test_oracle.py) and the reference's golden fixtures.

Bars: pyramids, selection tables, CSC lists and plans are
bit-exact; attention outputs and gradients within rel 1e-3 (fp32 inputs) or
2e-2 (bf16 inputs), measured as max|Δ|/max|ref| against the fp32 oracle run
on the same (bf16-widened) inputs.
"""
import numpy as np
import pytest
import torch

import paper_2512_16615_b200 as llsa
from oracle import Config, bf16_round, lse, rel_err, unit_inputs

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

DEV = "cuda"
# full-size bars (see test_full_size_tensor_core_path_matches_reference)
TOL_MAX, TOL_FRO, TOL_ROW, TOL_LSE = 2e-2, 1e-2, 6e-2, 1e-2


def T(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV, dtype)


def U32(t):
    return t.cpu().numpy().astype(np.uint32)


def vcfg(c: Config):
    return llsa.validate_config(llsa.LLSAConfig(c.n, c.d, c.block_size, c.top_k, c.levels,
                                                c.enrich_levels, c.softmax_scale,
                                                c.reweight_mode, c.safe_softmax))


# ---------------------------------------------------------------- compression
@pytest.mark.parametrize("rows,d,b,L,bf", [(64, 5, 4, 2, False), (81, 3, 3, 3, False),
                                           (4096, 64, 16, 2, True), (65536, 64, 16, 3, True),
                                           (1024, 32, 4, 4, False), (256, 6, 2, 7, True)])
def test_pyramid_bit_exact(oracle_c, rows, d, b, L, bf):
    x = oracle_c.gen_random(rows, d, 31337 + rows)
    if bf:
        x = bf16_round(x)
    got = llsa.build_pyramid(T(x, torch.bfloat16 if bf else torch.float32), b, L)
    want = oracle_c.build_pyramid(x, b, L)
    np.testing.assert_array_equal(got[0].cpu().numpy(), want)


def test_pyramid_kats(golden):
    for case in golden["kats"]["pyramid"]:
        x = T(np.array(case["x"], np.float32)[:, None])
        flat = llsa.build_pyramid(x, case["B"], case["L"])
        lv = llsa.pyramid_levels(flat, len(case["x"]), case["B"], case["L"])
        assert lv[case["level"] - 1][0, :, 0].cpu().tolist() == case["expect"]
    with pytest.raises(llsa.DivisibilityError):
        llsa.build_pyramid(T(np.ones((6, 1), np.float32)), 2, 2)


def test_pool_backward(oracle_c, golden):
    for case in golden["kats"]["pool_backward"]:
        out = llsa.pool_backward(T(np.array(case["g"], np.float32)[:, None]), case["B"],
                                 case["hops"])
        assert out[0, :, 0].cpu().tolist() == case["expect"]
    g = oracle_c.gen_random(16, 8, 5)
    for hops in (0, 1, 2):
        np.testing.assert_array_equal(llsa.pool_backward(T(g), 4, hops)[0].cpu().numpy(),
                                      oracle_c.pool_backward(g, 4, hops))


# ---------------------------------------------------------------- selection
def test_select_coarsest_bit_exact(oracle_c):
    for rows, cands, d, k, scale in ((12, 20, 6, 5, 0.33), (16, 16, 64, 8, 0.125),
                                     (256, 256, 64, 8, 0.125), (6, 8, 4, 8, 1.0),
                                     (64, 64, 64, 16, 0.125)):
        q = oracle_c.gen_random(rows, d, 21)
        kk = oracle_c.gen_random(cands, d, 22)
        got = llsa.select_coarsest(T(q), T(kk), k, scale)
        np.testing.assert_array_equal(U32(got[0]), oracle_c.select_coarsest(q, kk, k, scale))


def test_ties_break_to_smaller_index(golden, oracle_c):
    t = golden["kats"]["ties"]
    kk = np.tile(np.array(t["key_row"], np.float32), (t["key_rows"], 1))
    q = oracle_c.gen_random(t["q_rows"], t["d"], t["q_seed"])
    got = U32(llsa.select_coarsest(T(q), T(kk), t["top_k"], 1.0)[0])
    assert (got == np.array(t["expect_row"])).all()
    # exact-zero scores (all-zero pooled rows, e.g. padding) tie too
    z = np.zeros((32, 8), np.float32)
    got = U32(llsa.select_coarsest(T(z[:4]), T(z), 4, 0.125)[0])
    assert (got == np.arange(4)).all()


def test_select_level_bit_exact_and_validation(oracle_c):
    q = oracle_c.gen_random(16, 4, 5)
    kk = oracle_c.gen_random(16, 4, 6)
    parent = np.array([[0, 2], [1, 3], [0, 1], [2, 3]], np.uint32)
    got = llsa.select_level(T(q), T(kk), T(parent, torch.int32), 1, 3, 0.7, 4)
    np.testing.assert_array_equal(U32(got[0]), oracle_c.select_level(q, kk, parent, 1, 3, 0.7, 4))
    with pytest.raises(llsa.LevelError):
        llsa.select_level(T(q), T(kk), T(parent, torch.int32), 0, 2, 1.0, 4)
    with pytest.raises(llsa.ShapeMismatch):
        llsa.select_level(T(q[:12]), T(kk), T(parent, torch.int32), 1, 2, 1.0, 4)
    with pytest.raises(llsa.TopKError):
        llsa.select_level(T(q), T(kk), T(parent, torch.int32), 1, 9, 1.0, 4)
    bad = parent.copy()
    bad[1, 1] = 4
    llsa.select_level(T(q), T(kk), T(bad, torch.int32), 1, 2, 1.0, 4)
    with pytest.raises(llsa.IndexOutOfRange):
        llsa.sync_status()


def test_select_level_unsorted_parent_rows_match_oracle(oracle_c):
    # topk_row ends with std::sort (selection.cpp:37): the output rows ascend
    # whatever order the parent row lists its blocks in.  d = 64, B = 16 runs
    # the fast kernel; d = 4, B = 4 the generic one.
    rng = np.random.default_rng(5)
    for rows, d, b, k in ((4096, 64, 16, 8), (64, 4, 4, 3)):
        kb = rows // b
        q = oracle_c.gen_random(rows, d, 50)
        kk = oracle_c.gen_random(rows, d, 51)
        parent = np.stack([rng.permutation(kb)[:k] for _ in range(rows // b)]).astype(np.uint32)
        got = llsa.select_level(T(q), T(kk), T(parent, torch.int32), 1, k, 0.125, b)
        want = oracle_c.select_level(q, kk, parent, 1, k, 0.125, b)
        np.testing.assert_array_equal(U32(got[0]), want)
        assert (np.diff(U32(got[0]).astype(np.int64), axis=1) > 0).all()


@pytest.mark.parametrize("name", ["c1_n4096_L1", "c1_n4096_L2", "c2_n16384_L2",
                                  "c3_n65536_L3", "c3p_n65536_L2"])
def test_hierarchical_topk_matches_reference_tables(golden, oracle_c, name):
    g = golden["tables"]
    n, d, b, k, L, le, seed = (int(x) for x in g[f"{name}/cfg"])
    cfg = vcfg(Config(n, d, b, k, L, le))
    q, kk = (bf16_round(oracle_c.gen_random(n, d, seed + i)) for i in range(2))
    pq = llsa.build_pyramid(T(q, torch.bfloat16), b, L)
    pk = llsa.build_pyramid(T(kk, torch.bfloat16), b, L)
    tables = llsa.hierarchical_topk(pq, pk, cfg)
    np.testing.assert_array_equal(U32(tables[0]), g[f"{name}/tables"])


def test_hierarchical_topk_batched_units(oracle_c):
    cfg = Config(4096, 64, 16, 8, 2, 2)
    qs, ks, want = [], [], []
    for u in range(3):
        q, kk, _, _ = unit_inputs(cfg, u, backend=oracle_c)
        qs.append(q)
        ks.append(kk)
        want.append(oracle_c.run(cfg, q, kk, kk).tables)
    vc = vcfg(cfg)
    pq = llsa.build_pyramid(T(np.stack(qs), torch.bfloat16), 16, 2)
    pk = llsa.build_pyramid(T(np.stack(ks), torch.bfloat16), 16, 2)
    got = U32(llsa.hierarchical_topk(pq, pk, vc))
    for u in range(3):
        np.testing.assert_array_equal(got[u], want[u])


# ---------------------------------------------------------------- transpose
def test_transpose_kats(golden):
    for case in golden["kats"]["transpose"]:
        idx = np.array(case["idx"], np.int32).reshape(case["rows"], case["k"])
        offs, flat = llsa.transpose_indices(T(idx, torch.int32), case["key_blocks"])
        assert offs[0].cpu().tolist() == case["offsets"]
        assert flat[0].cpu().tolist() == case["flat"]


def test_transpose_random_tables_match_oracle(oracle_c):
    # acceptance A4 (P/tests/acceptance.cpp:168-217): random tables, exact
    rng = np.random.default_rng(2024)
    for _ in range(60):
        qb, kb = int(rng.integers(1, 65)), int(rng.integers(1, 65))
        k = int(rng.integers(1, min(8, kb) + 1))
        idx = np.stack([np.sort(rng.permutation(kb)[:k]) for _ in range(qb)]).astype(np.uint32)
        o, f = llsa.transpose_indices(T(idx.astype(np.int32), torch.int32), kb)
        wo, wf = oracle_c.transpose(idx, kb)
        np.testing.assert_array_equal(U32(o[0]), wo)
        np.testing.assert_array_equal(U32(f[0]), wf)


def test_transpose_degenerate_long_segment(oracle_c):
    # every row picks the same blocks (constant keys → tie-break): segments = T
    idx = np.tile(np.arange(8, dtype=np.uint32), (4096, 1))
    o, f = llsa.transpose_indices(T(idx.astype(np.int32), torch.int32), 4096)
    wo, wf = oracle_c.transpose(idx, 4096)
    np.testing.assert_array_equal(U32(o[0]), wo)
    np.testing.assert_array_equal(U32(f[0]), wf)


def test_handle_skewed_selection_long_segments(oracle_c):
    # constant keys: every score of a row ties, so every query block picks the
    # K lowest blocks (topk_row's tie-break) and each picked key block's CSC
    # segment holds every query block of its level (4096/256/16 entries at
    # N = 65536, L = 3): the transpose's CTA-sort path, then the backward
    # walks those hot segments
    cfg = Config(16384, 64, 16, 8, 2, 2)
    q, _, v, dO = unit_inputs(cfg, 0, bf16=True, backend=oracle_c)
    k = np.full_like(q, 0.5)
    ref = oracle_c.run(cfg, q, k, v, dO)
    h = llsa.LLSAHandle(llsa.LLSAConfig(cfg.n, 64, 16, 8, 2, 2), 1, torch.bfloat16)
    tq, tk, tv, tdo = (T(a, torch.bfloat16)[None] for a in (q, k, v, dO))
    out = h.forward(tq, tk, tv)
    dq, dk, dv = h.backward(tdo, tq, tk, tv, out)
    llsa.sync_status()
    np.testing.assert_array_equal(U32(h.view("tables"))[0], ref.tables)
    np.testing.assert_array_equal(U32(h.view("csc_offsets"))[0], ref.csc_offsets)
    np.testing.assert_array_equal(U32(h.view("csc_flat"))[0], ref.csc_flat)
    for name, got, want in (("out", out, ref.out), ("dq", dq, ref.dq), ("dk", dk, ref.dk),
                            ("dv", dv, ref.dv)):
        e = rel_err(got[0].cpu().numpy(), want)
        assert e["max_rel"] <= 2e-2, (name, e)
    # and at N = 65536 through the transpose alone (segments up to 4096 long)
    cfg3 = Config(65536, 64, 16, 8, 3, 3)
    vc = vcfg(cfg3)
    tables = np.concatenate([np.tile(np.arange(8, dtype=np.int32), rows)
                             for rows in cfg3.table_rows()])
    offs, flat = llsa.transpose_all(T(tables, torch.int32)[None], vc)
    for l, t in enumerate(cfg3.split_tables(tables.astype(np.uint32))):
        wo, wf = oracle_c.transpose(t, cfg3.level_blocks(l))
        lo = sum(cfg3.level_blocks(j) + 1 for j in range(l))
        lf = sum(cfg3.level_blocks(j) * 8 for j in range(l))
        np.testing.assert_array_equal(U32(offs[0])[lo:lo + wo.size], wo)
        np.testing.assert_array_equal(U32(flat[0])[lf:lf + wf.size], wf)


def test_transpose_out_of_range_flags():
    idx = np.array([[0], [5]], np.int32)
    llsa.transpose_indices(T(idx, torch.int32), 4)
    with pytest.raises(llsa.IndexOutOfRange):
        llsa.sync_status()


# ---------------------------------------------------------------- forward / backward
SMALL = [Config(256, 8, 4, 2, 2, 2), Config(256, 8, 4, 2, 2, 2, reweight_mode=1),
         Config(128, 8, 4, 2, 2, 0), Config(128, 8, 4, 2, 2, 1),
         Config(64, 8, 4, 16, 1, 0), Config(256, 8, 4, 2, 2, 2, safe_softmax=False),
         Config(1024, 16, 4, 4, 3, 3), Config(512, 33, 8, 3, 1, 1),
         Config(4096, 64, 16, 8, 1, 1), Config(4096, 64, 16, 8, 2, 2)]


def _staged(oracle_c, cfg: Config, seed: int, bf: bool):
    q, k, v, dO = (oracle_c.gen_random(cfg.n, cfg.d, seed + i) for i in range(4))
    if bf:
        q, k, v, dO = (bf16_round(a) for a in (q, k, v, dO))
    ref = oracle_c.run(cfg, q, k, v, dO)
    dt = torch.bfloat16 if bf else torch.float32
    vc = vcfg(cfg)
    tq, tk, tv, tdo = (T(a, dt) for a in (q, k, v, dO))
    pk = llsa.build_pyramid(tk, cfg.block_size, cfg.levels)
    pv = llsa.build_pyramid(tv, cfg.block_size, cfg.levels)
    pq = llsa.build_pyramid(tq, cfg.block_size, cfg.levels)
    tables = llsa.hierarchical_topk(pq, pk, vc)
    return ref, vc, (tq, tk, tv, tdo), pk, pv, tables


@pytest.mark.parametrize("cfg", SMALL, ids=lambda c: f"n{c.n}d{c.d}B{c.block_size}L{c.levels}"
                         f"e{c.enrich_levels}m{c.reweight_mode}s{int(c.safe_softmax)}")
@pytest.mark.parametrize("bf", [False, True])
def test_staged_path_matches_oracle(oracle_c, cfg, bf, deterministic):
    # bf16 inputs at d = 64, B = 16 (safe softmax) run the tensor-core kernels
    # behind the staged C ABI (the bf16 bar); everything else the fp32 SIMT
    # kernels (rounding-level agreement)
    tc = bf and cfg.d == 64 and cfg.block_size == 16 and cfg.safe_softmax
    ref, vc, (tq, tk, tv, tdo), pk, pv, tables = _staged(oracle_c, cfg, 100 + cfg.n, bf)
    np.testing.assert_array_equal(U32(tables[0]), ref.tables)
    lv, bl, w = llsa.build_plan(tables, vc)
    np.testing.assert_array_equal(U32(lv[0]).reshape(-1), ref.plan_level)
    np.testing.assert_array_equal(U32(bl[0]).reshape(-1), ref.plan_block)
    np.testing.assert_array_equal(w[0].cpu().numpy().reshape(-1), ref.plan_weight)
    st = llsa.llsa_forward(tq, tk, tv, pk, pv, tables, vc)
    tol = 2e-2 if tc else 1e-4   # fp32 math on identical inputs: rounding-level agreement
    assert rel_err(st.output[0].cpu().numpy(), ref.out)["max_rel"] <= tol
    np.testing.assert_allclose(lse(st.row_max[0].cpu().numpy(), st.row_denom[0].cpu().numpy()),
                               lse(ref.row_max, ref.row_denom),
                               rtol=1e-5, atol=TOL_LSE if tc else 1e-4)
    tr = llsa.transpose_all(tables, vc)
    np.testing.assert_array_equal(U32(tr[0][0]), ref.csc_offsets)
    np.testing.assert_array_equal(U32(tr[1][0]), ref.csc_flat)
    dq, dk, dv = llsa.llsa_backward(tdo, st, tq, tk, tv, pk, pv, tables, tr, vc)
    llsa.sync_status()
    for name, got, want in (("dq", dq, ref.dq), ("dk", dk, ref.dk), ("dv", dv, ref.dv)):
        e = rel_err(got[0].cpu().numpy(), want)
        assert e["max_rel"] <= (2e-2 if tc else 1e-3), (name, e)
    # kv_backward (CSC lists only; the tensor-core path rebuilds the tables)
    # runs the same kernels: bit-identical dk, dv
    dk2, dv2 = llsa.kv_backward(tdo, st, tq, tk, tv, pk, pv, tr, vc)
    llsa.sync_status()
    assert torch.equal(dk2, dk) and torch.equal(dv2, dv)
    # the mask-based baseline (oracle.cpp:365-501) finds the same key→query
    # lists through dense block masks and runs the same kernels: identical
    dk3, dv3 = llsa.mask_kv_backward(tdo, st, tq, tk, tv, pk, pv, tables, vc)
    llsa.sync_status()
    assert torch.equal(dk3, dk) and torch.equal(dv3, dv)


def test_forward_overflow_without_rescaling_raises():
    # P/tests/test_attention.cpp:180-223
    q = np.full((16, 8), 300.0, np.float32)
    k = np.ones((16, 8), np.float32)
    from oracle import OracleC
    v = OracleC().gen_random(16, 8, 31)
    for safe, raises in ((False, True), (True, False)):
        vc = llsa.validate_config(llsa.LLSAConfig(16, 8, 4, 2, 1, 0, safe_softmax=safe))
        pq, pk, pv = (llsa.build_pyramid(T(a), 4, 1) for a in (q, k, v))
        tables = llsa.hierarchical_topk(pq, pk, vc)
        if raises:
            with pytest.raises(llsa.NonFiniteError):
                llsa.llsa_forward(T(q), T(k), T(v), pk, pv, tables, vc)
        else:
            st = llsa.llsa_forward(T(q), T(k), T(v), pk, pv, tables, vc)
            assert torch.isfinite(st.output).all()


def test_zero_cotangent_gives_zero_gradients(oracle_c):
    cfg = Config(64, 4, 4, 2, 2, 2)
    ref, vc, (tq, tk, tv, tdo), pk, pv, tables = _staged(oracle_c, cfg, 3, False)
    st = llsa.llsa_forward(tq, tk, tv, pk, pv, tables, vc)
    tr = llsa.transpose_all(tables, vc)
    grads = llsa.llsa_backward(torch.zeros_like(tdo), st, tq, tk, tv, pk, pv, tables, tr, vc)
    for g in grads:
        assert (g == 0).all()


# ---------------------------------------------------------------- fused handle
@pytest.mark.parametrize("cfg,bf", [(Config(4096, 64, 16, 8, 1, 1), False),
                                    (Config(4096, 64, 16, 8, 2, 2), True),
                                    (Config(16384, 64, 16, 8, 2, 2), True),
                                    (Config(16384, 64, 16, 8, 2, 2, reweight_mode=1), True),
                                    (Config(16384, 64, 16, 8, 2, 0), True),
                                    (Config(65536, 64, 16, 8, 3, 3), True)])
def test_handle_path_matches_oracle(oracle_c, reference, cfg, bf, deterministic):
    # the single-threaded C restatement up to C2; the multi-threaded compiled
    # reference at N = 65536 (forward and backward on both units)
    units = 2
    import os
    reference.set_threads(os.cpu_count() or 1)
    be = oracle_c if cfg.n <= 16384 else reference
    ins = [unit_inputs(cfg, u, bf16=bf, backend=be) for u in range(units)]
    want_bwd = True
    refs = [be.run(cfg, q, k, v, dO) for q, k, v, dO in ins]
    dt = torch.bfloat16 if bf else torch.float32
    q, k, v, dO = (T(np.stack([i[j] for i in ins]), dt) for j in range(4))
    h = llsa.LLSAHandle(llsa.LLSAConfig(cfg.n, cfg.d, cfg.block_size, cfg.top_k, cfg.levels,
                                        cfg.enrich_levels,
                                        reweight_mode=cfg.reweight_mode), units, dt)
    out = h.forward(q, k, v)
    tol = 2e-2 if bf else 1e-3
    tables = U32(h.view("tables"))
    for u in range(units):
        np.testing.assert_array_equal(tables[u], refs[u].tables)
        e = rel_err(out[u].cpu().numpy(), refs[u].out)
        assert e["max_rel"] <= tol and e["p99_row"] <= 2.5 * tol, ("out", u, e)
        g_lse = lse(h.view("row_max")[u].cpu().numpy(), h.view("row_denom")[u].cpu().numpy())
        assert np.abs(g_lse - lse(refs[u].row_max, refs[u].row_denom)).max() <= \
            (TOL_LSE if bf else 1e-4)
    if want_bwd:
        dq, dk, dv = h.backward(dO, q, k, v, out)
        llsa.sync_status()
        for u in range(units):
            for name, got, want in (("dq", dq, refs[u].dq), ("dk", dk, refs[u].dk),
                                    ("dv", dv, refs[u].dv)):
                e = rel_err(got[u].cpu().numpy(), want)
                assert e["max_rel"] <= tol and e["p99_row"] <= 2.5 * tol, (name, u, e)
        # determinism: a second run is bitwise identical
        out2 = h.forward(q, k, v)
        g2 = h.backward(dO, q, k, v, out2)
        assert torch.equal(out, out2)
        for a, b in zip((dq, dk, dv), g2):
            assert torch.equal(a, b)


# ------------------------------------- full-size tcgen05 path vs the reference
# The compiled, unmodified reference (oracle/_ref/libllsa_ref32.so, the f32
# build, multi-threaded) is the checker at every BASELINE size: C2, C3 (K = 8
# and 16, L_e = 3 and 1, ScaleKV and LogitBias), C3' (L = 2) and all six C5
# points (N = 262144, K = 4 / 8 / 16, L_e = 3 and 0; L = 4 is inadmissible at
# N = 262144).  Inputs are the reference's own gen_random
# streams rounded to bf16; the reference runs on the same
# widened values.  Bars: every selection table bit-exact; O, dq, dk, dv within
# 2e-2 of max|ref| AND 1e-2 relative Frobenius AND 6e-2 for the 99th
# percentile of the row-relative error (a missing or mis-weighted coarse
# contribution in a low-magnitude row shows up in the last two; the worst row
# is logged, not asserted: dq rows whose coarse terms cancel carry the bf16
# rounding of K'·gain, see DESIGN.md §3 Precision); the LSE m + ln(denom) from the handle's row_max /
# row_denom within 1e-2 absolute (LSE values are ~20-40 here: the tensor-core
# row sums add P after its bf16 rounding, the same P that multiplies V).  The measured errors are appended to
# $LLSA_PARITY_LOG (profiles/r2_parity.json keeps a round's run).
REF_CASES = [
    ("C2", Config(16384, 64, 16, 8, 2, 2)),
    ("C3", Config(65536, 64, 16, 8, 3, 3)),
    ("C3-K16", Config(65536, 64, 16, 16, 3, 3)),
    ("C3-Le1", Config(65536, 64, 16, 8, 3, 1)),
    ("C3-LogitBias", Config(65536, 64, 16, 8, 3, 3, reweight_mode=1)),
    ("C3p-L2", Config(65536, 64, 16, 8, 2, 2)),
    ("C5-K4", Config(262144, 64, 16, 4, 3, 3)),
    ("C5-K8", Config(262144, 64, 16, 8, 3, 3)),
    ("C5-K16", Config(262144, 64, 16, 16, 3, 3)),
    ("C5-K4-Le0", Config(262144, 64, 16, 4, 3, 0)),
    ("C5-K8-Le0", Config(262144, 64, 16, 8, 3, 0)),
    ("C5-K16-Le0", Config(262144, 64, 16, 16, 3, 0)),
]

def _log_parity(rec: dict) -> None:
    import json
    import os
    path = os.environ.get("LLSA_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("name,cfg", REF_CASES, ids=[c[0] for c in REF_CASES])
def test_full_size_tensor_core_path_matches_reference(reference, name, cfg):
    import os
    import time
    reference.set_threads(os.cpu_count() or 1)
    q, k, v, dO = unit_inputs(cfg, 0, bf16=True, backend=reference)
    t0 = time.perf_counter()
    ref = reference.run(cfg, q, k, v, dO)
    ref_s = time.perf_counter() - t0
    lc = llsa.LLSAConfig(cfg.n, 64, 16, cfg.top_k, cfg.levels, cfg.enrich_levels,
                         reweight_mode=cfg.reweight_mode)
    h = llsa.LLSAHandle(lc, 1, torch.bfloat16)
    assert h.uses_tensor_cores
    tq, tk, tv, tdo = (T(a, torch.bfloat16)[None] for a in (q, k, v, dO))
    out = h.forward(tq, tk, tv)
    dq, dk, dv = h.backward(tdo, tq, tk, tv, out)
    llsa.sync_status()
    rec = {"case": name, "n": cfg.n, "top_k": cfg.top_k, "levels": cfg.levels,
           "enrich_levels": cfg.enrich_levels,
           "mode": "LogitBias" if cfg.reweight_mode else "ScaleKV",
           "reference_s": round(ref_s, 3), "reference_threads": reference.threads()}
    got_tables = U32(h.view("tables"))[0]
    diff_rows = 0
    for l, (gt, wt) in enumerate(zip(cfg.split_tables(got_tables),
                                     cfg.split_tables(ref.tables))):
        diff_rows += int((gt != wt).any(axis=1).sum())
    rec["table_rows_differing"] = diff_rows
    for nm, got, want in (("out", out, ref.out), ("dq", dq, ref.dq), ("dk", dk, ref.dk),
                          ("dv", dv, ref.dv)):
        rec[nm] = rel_err(got[0].cpu().numpy(), want)
    g_lse = lse(h.view("row_max")[0].cpu().numpy(), h.view("row_denom")[0].cpu().numpy())
    rec["lse_max_abs"] = float(np.abs(g_lse - lse(ref.row_max, ref.row_denom)).max())
    _log_parity(rec)
    assert diff_rows == 0, rec
    np.testing.assert_array_equal(got_tables, ref.tables)
    for nm in ("out", "dq", "dk", "dv"):
        e = rec[nm]
        assert e["max_rel"] <= TOL_MAX and e["fro"] <= TOL_FRO and e["p99_row"] <= TOL_ROW, \
            (nm, rec)
    assert rec["lse_max_abs"] <= TOL_LSE, rec


# The persistent tcgen05 kernels walk (unit, tile) work items; a multi-unit
# handle must give every unit exactly what a one-unit handle gives it.
@pytest.mark.parametrize("n,L", [(16384, 2), (65536, 3)])
def test_multi_unit_handle_is_per_unit_exact(n, L, deterministic):
    units = 3
    g = torch.Generator(device="cuda").manual_seed(21)
    q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
                   for _ in range(4))
    lc = llsa.LLSAConfig(n, 64, 16, 8, L, L)
    hm = llsa.LLSAHandle(lc, units, torch.bfloat16)
    assert hm.uses_tensor_cores
    out = hm.forward(q, k, v)
    grads = hm.backward(dO, q, k, v, out)
    h1 = llsa.LLSAHandle(lc, 1, torch.bfloat16)
    for u in range(units):
        sl = slice(u, u + 1)
        o1 = h1.forward(q[sl], k[sl], v[sl])
        g1 = h1.backward(dO[sl], q[sl], k[sl], v[sl], o1)
        assert torch.equal(out[sl], o1), u
        for a, b in zip(grads, g1):
            assert torch.equal(a[sl], b), u
    llsa.sync_status()


@pytest.mark.parametrize("n,L", [(16384, 2), (65536, 3)])
def test_staged_tensor_core_path_equals_handle(n, L, deterministic):
    # the reference-shaped staged C ABI (bf16) runs the handle's kernels:
    # tables, CSC lists, forward and backward bit-identical, 2 units
    units = 2
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
                   for _ in range(4))
    cfg = llsa.LLSAConfig(n, 64, 16, 8, L, L)
    vc = llsa.validate_config(cfg)
    h = llsa.LLSAHandle(cfg, units)
    o = h.forward(q, k, v)
    grads = h.backward(dO, q, k, v, o)
    pq, pk, pv = (llsa.build_pyramid(t, 16, L) for t in (q, k, v))
    tables = llsa.hierarchical_topk(pq, pk, vc)
    assert torch.equal(tables.view(-1), h.view("tables").view(-1))
    st = llsa.llsa_forward(q, k, v, pk, pv, tables, vc)
    assert torch.equal(st.output, o)
    tr = llsa.transpose_all(tables, vc)
    assert torch.equal(tr[0].view(-1), h.view("csc_offsets").view(-1))
    assert torch.equal(tr[1].view(-1), h.view("csc_flat").view(-1))
    sg = llsa.llsa_backward(dO, st, q, k, v, pk, pv, tables, tr, vc)
    for a, b in zip(sg, grads):
        assert torch.equal(a, b)
    dk, dv = llsa.kv_backward(dO, st, q, k, v, pk, pv, tr, vc)
    llsa.sync_status()
    assert torch.equal(dk, grads[1]) and torch.equal(dv, grads[2])


# -------------------------------------------- randomized sweep vs the reference
def _random_configs(count, seed):
    """Admissible configs drawn like the reference's own constraints
    (config.cpp:54-125): n = B^(L+1)·m, K <= n / B^L, L_e <= L.  Every third
    one has the tensor-core shape (d = 64, B = 16, bf16 inputs)."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        tc = len(out) % 3 == 2
        b = 16 if tc else int(rng.choice([2, 4, 8, 16]))
        L = int(rng.integers(1, 3 if tc else 4))
        m = int(rng.integers(1, 5))
        n = b ** (L + 1) * m
        if n > 16384 or n < 16:
            continue
        kmax = n // b ** L
        k = int(rng.integers(1, min(kmax, 16) + 1))
        d = 64 if tc else int(rng.choice([8, 16, 33, 64]))
        le = int(rng.integers(0, L + 1))
        mode = int(rng.integers(0, 2))
        out.append(Config(n, d, b, k, L, le, reweight_mode=mode))
    return out


@pytest.mark.parametrize("cfg", _random_configs(24, 2026),
                         ids=lambda c: f"n{c.n}d{c.d}B{c.block_size}K{c.top_k}L{c.levels}"
                         f"e{c.enrich_levels}m{c.reweight_mode}")
def test_random_configs_match_reference(reference, cfg):
    # the handle (any shape: SIMT kernels in fp32, tensor cores for bf16 at
    # d = 64, B = 16) against the compiled reference on its own inputs
    bf = cfg.d == 64 and cfg.block_size == 16
    q, k, v, dO = unit_inputs(cfg, 0, seed=7, bf16=bf, backend=reference)
    ref = reference.run(cfg, q, k, v, dO)
    dt = torch.bfloat16 if bf else torch.float32
    h = llsa.LLSAHandle(llsa.LLSAConfig(cfg.n, cfg.d, cfg.block_size, cfg.top_k, cfg.levels,
                                        cfg.enrich_levels, reweight_mode=cfg.reweight_mode),
                        1, dt)
    tq, tk, tv, tdo = (T(a, dt)[None] for a in (q, k, v, dO))
    out = h.forward(tq, tk, tv)
    dq, dk, dv = h.backward(tdo, tq, tk, tv, out)
    llsa.sync_status()
    np.testing.assert_array_equal(U32(h.view("tables"))[0], ref.tables)
    np.testing.assert_array_equal(U32(h.view("csc_offsets"))[0], ref.csc_offsets)
    np.testing.assert_array_equal(U32(h.view("csc_flat"))[0], ref.csc_flat)
    tol = 2e-2 if h.uses_tensor_cores else 1e-3
    for name, got, want in (("out", out, ref.out), ("dq", dq, ref.dq), ("dk", dk, ref.dk),
                            ("dv", dv, ref.dv)):
        e = rel_err(got[0].cpu().numpy(), want)
        assert e["max_rel"] <= tol and e["fro"] <= tol, (name, e)


# The default coarse dK'/dV' path adds every (row, group) item into the level
# slots with fp32 TMA reductions (unordered); LLSA_DETERMINISTIC=1 writes raw
# partials and sums them in CSC order.  Same math, different fp32 summation
# order: dq and the output identical, dk / dv equal to fp32 rounding.
@pytest.mark.parametrize("n,L,Le", [(16384, 2, 2), (65536, 3, 3), (65536, 2, 2),
                                    (65536, 3, 1)])
def test_reduce_add_rows_match_ordered_sum(monkeypatch, n, L, Le):
    units = 2
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
                   for _ in range(4))
    cfg = llsa.LLSAConfig(n, 64, 16, 8, L, Le)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("LLSA_DETERMINISTIC", mode)
        h = llsa.LLSAHandle(cfg, units)
        out = h.forward(q, k, v)
        res[mode] = (out,) + tuple(h.backward(dO, q, k, v, out))
    llsa.sync_status()
    a, b = res["0"], res["1"]
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    for x, y in zip(a[2:], b[2:]):
        assert float((x - y).abs().max()) <= 1e-5 * float(y.abs().max())


# The largest BASELINE batches in one handle — C4's per-GPU batch (128 units
# of N = 65536) and C5's 16 units of N = 262144: every index, TMA coordinate
# and work-item decode at full size.  Sampled units must equal a one-unit
# handle's results bit for bit (ordered mode).
@pytest.mark.parametrize("units,n,L,K", [(128, 65536, 3, 8), (16, 262144, 3, 8),
                                         (128, 16384, 2, 8), (16, 262144, 3, 16)])
def test_largest_batches_match_single_unit_handle(deterministic, units, n, L, K):
    g = torch.Generator(device="cuda").manual_seed(44)
    q, k, v, dO = (torch.randn(units, n, 64, device="cuda", generator=g).to(torch.bfloat16)
                   for _ in range(4))
    lc = llsa.LLSAConfig(n, 64, 16, K, L, L)
    hm = llsa.LLSAHandle(lc, units, torch.bfloat16)
    out = hm.forward(q, k, v, out_dtype=torch.bfloat16)
    grads = hm.backward(dO, q, k, v, out)
    llsa.sync_status()
    h1 = llsa.LLSAHandle(lc, 1, torch.bfloat16)
    for u in sorted({0, units // 2 + 5, units - 1}):
        sl = slice(u, u + 1)
        o1 = h1.forward(q[sl], k[sl], v[sl], out_dtype=torch.bfloat16)
        g1 = h1.backward(dO[sl], q[sl], k[sl], v[sl], o1)
        assert torch.equal(out[sl], o1), u
        for a, b in zip(grads, g1):
            assert torch.equal(a[sl], b), u
    llsa.sync_status()

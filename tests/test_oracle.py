"""Pins the C restatement (oracle/llsa_oracle.c) before anything trusts it.

1. Known-answer tests transcribed from the reference's unit tests
   (tests/golden/kats.json, file:line per entry).
2. Bit-exact equality with fixtures produced by the reference library itself
   (tests/golden/ref_*.npz, see tests/golden/make_golden.py).
3. Where oracle/_ref is built, bit-exact equality with the live reference on
   fresh seeds (f32 build) and closeness to the f64 build.
"""
import hashlib

import numpy as np
import pytest

from oracle import Config, OracleC, bf16_round, rel_err


def _cfg(row):
    n, d, b, k, L, le, mode, safe = (int(x) for x in row[:8])
    return Config(n, d, b, k, L, le, reweight_mode=mode, safe_softmax=bool(safe))


def test_max_levels_kats(oracle_c, golden):
    for n, b, want in golden["kats"]["max_levels"]["cases"]:
        assert oracle_c.max_levels(n, b) == want


def test_effective_block_count_kats(oracle_c, golden):
    for (n, d, b, k, L, le), want in golden["kats"]["effective_block_count"]["cases"]:
        code, _, eff = oracle_c.validate(Config(n, d, b, k, L, le))
        assert code == 0 and eff == want


def test_validate_kats(oracle_c, golden):
    for (n, d, b, k, L, le), want in golden["kats"]["validate"]["cases"]:
        assert oracle_c.validate(Config(n, d, b, k, L, le))[0] == want, (n, d, b, k, L, le)
    bad = Config(64, 4, 4, 1, 1, 0, softmax_scale=-1.0)
    assert oracle_c.validate(bad)[0] == 1
    bad.softmax_scale = float("nan")
    assert oracle_c.validate(bad)[0] == 1
    assert oracle_c.validate(Config(64, 16, 4, 2, 1, 0))[1] == 0.25


def test_pyramid_kats(oracle_c, golden):
    for case in golden["kats"]["pyramid"]:
        x = np.array(case["x"], np.float32)[:, None]
        flat = oracle_c.build_pyramid(x, case["B"], case["L"])
        lv = Config(len(case["x"]), 1, case["B"], 1, case["L"], 0).split_pyramid(flat)
        np.testing.assert_array_equal(lv[case["level"] - 1][:, 0], case["expect"])


def test_pool_backward_kats(oracle_c, golden):
    for case in golden["kats"]["pool_backward"]:
        out = oracle_c.pool_backward(np.array(case["g"], np.float32)[:, None], case["B"],
                                     case["hops"])
        np.testing.assert_array_equal(out[:, 0], case["expect"])
    g = oracle_c.gen_random(8, 2, 3)
    np.testing.assert_array_equal(oracle_c.pool_backward(g, 2, 0), g)


def test_pool_backward_is_adjoint(oracle_c):
    # P/tests/test_pyramid.cpp:113-132
    x = oracle_c.gen_random(64, 4, 11)
    flat = oracle_c.build_pyramid(x, 4, 2)
    lv = Config(64, 4, 4, 1, 2, 0).split_pyramid(flat)
    for hops in (1, 2):
        y = oracle_c.gen_random(lv[hops - 1].shape[0], 4, 100 + hops)
        yt = oracle_c.pool_backward(y, 4, hops)
        lhs = float((lv[hops - 1].astype(np.float64) * y).sum())
        rhs = float((x.astype(np.float64) * yt).sum())
        assert abs(lhs - rhs) <= 1e-5 * (1 + abs(lhs))


def test_transpose_kats(oracle_c, golden):
    for case in golden["kats"]["transpose"]:
        idx = np.array(case["idx"], np.uint32).reshape(case["rows"], case["k"])
        offs, flat = oracle_c.transpose(idx, case["key_blocks"])
        assert offs.tolist() == case["offsets"]
        assert flat.tolist() == case["flat"]


def test_transpose_rejects_out_of_range(oracle_c):
    from oracle import OracleError
    with pytest.raises(OracleError) as e:
        oracle_c.transpose(np.array([[0], [5]], np.uint32), 4)
    assert e.value.code == 6


def test_ties_break_to_smaller_index(oracle_c, golden):
    t = golden["kats"]["ties"]
    k = np.tile(np.array(t["key_row"], np.float32), (t["key_rows"], 1))
    q = oracle_c.gen_random(t["q_rows"], t["d"], t["q_seed"])
    out = oracle_c.select_coarsest(q, k, t["top_k"], 1.0)
    for row in out:
        assert row.tolist() == t["expect_row"]


def test_keep_all_is_identity(oracle_c):
    # P/tests/test_selection.cpp:83-91
    q, k = oracle_c.gen_random(6, 4, 1), oracle_c.gen_random(8, 4, 2)
    out = oracle_c.select_coarsest(q, k, 8, 1.0)
    assert (out == np.arange(8)).all()


@pytest.mark.parametrize("name", ["n256_scalekv", "n256_logitbias", "n128_noenrich",
                                  "n128_partial", "n64_dense", "n256_unsafe",
                                  "n1024_d64_b16"])
def test_oracle_matches_reference_fixture_bitwise(oracle_c, golden, name):
    g = golden["small"]
    row = g[f"{name}/cfg"]
    cfg = _cfg(row)
    seed, bf = int(row[8]), bool(row[9])
    arrs = [oracle_c.gen_random(cfg.n, cfg.d, seed + i) for i in range(4)]
    if bf:
        arrs = [bf16_round(a) for a in arrs]
    r = oracle_c.run(cfg, *arrs)
    for key in ("pyr_q", "pyr_k", "pyr_v", "tables", "out", "row_max", "row_denom",
                "csc_offsets", "csc_flat", "dq", "dk", "dv", "plan_level", "plan_block",
                "plan_weight"):
        np.testing.assert_array_equal(getattr(r, key).reshape(-1),
                                      g[f"{name}/{key}"].reshape(-1), err_msg=key)
    assert r.checksum == int(g[f"{name}/checksum"][0])


@pytest.mark.parametrize("name", ["c1_n4096_L1", "c1_n4096_L2", "c2_n16384_L2",
                                  "c3_n65536_L3", "c3p_n65536_L2"])
def test_oracle_selection_matches_reference_tables(oracle_c, golden, name):
    g = golden["tables"]
    n, d, b, k, L, le, seed = (int(x) for x in g[f"{name}/cfg"])
    cfg = Config(n, d, b, k, L, le)
    q, kk = (bf16_round(oracle_c.gen_random(n, d, seed + i)) for i in range(2))
    pq = oracle_c.build_pyramid(q, b, L)
    pk = oracle_c.build_pyramid(kk, b, L)
    assert hashlib.sha256(pk.tobytes()).hexdigest() == str(g[f"{name}/pyr_k_sha256"][0])
    import ctypes as C
    tables = np.zeros(sum(cfg.table_rows()) * k, np.uint32)
    macs = C.c_uint64(0)
    code = oracle_c.lib.oracle_hierarchical_topk(C.byref(cfg.raw()), pq, pk, tables,
                                                 C.byref(macs))
    assert code == 0
    np.testing.assert_array_equal(tables, g[f"{name}/tables"])
    if f"{name}/csc_offsets" in g:
        offs_all, flat_all = [], []
        for l, t in enumerate(cfg.split_tables(tables)):
            o, f = oracle_c.transpose(t, cfg.level_blocks(l))
            offs_all.append(o)
            flat_all.append(f)
        np.testing.assert_array_equal(np.concatenate(offs_all), g[f"{name}/csc_offsets"])
        np.testing.assert_array_equal(np.concatenate(flat_all), g[f"{name}/csc_flat"])


@pytest.mark.parametrize("cfg,seed", [
    (Config(256, 8, 4, 2, 2, 2), 101),
    (Config(256, 8, 4, 3, 3, 3, reweight_mode=1), 102),
    (Config(512, 16, 8, 4, 1, 0), 103),
    (Config(4096, 64, 16, 8, 2, 1), 104),
])
def test_oracle_matches_live_reference(oracle_c, reference, cfg, seed):
    q, k, v, dO = (reference.gen_random(cfg.n, cfg.d, seed + i) for i in range(4))
    assert np.array_equal(q, oracle_c.gen_random(cfg.n, cfg.d, seed))
    a = oracle_c.run(cfg, q, k, v, dO)
    b = reference.run(cfg, q, k, v, dO)
    for key in ("tables", "out", "row_max", "row_denom", "csc_flat", "dq", "dk", "dv"):
        np.testing.assert_array_equal(getattr(a, key), getattr(b, key), err_msg=key)


def test_oracle_close_to_f64_reference(oracle_c):
    from oracle import REF_SO, Reference
    import os
    if not os.path.exists(REF_SO[64]):
        pytest.skip("f64 reference not built")
    r64 = Reference(64)
    cfg = Config(1024, 16, 4, 4, 3, 3)
    q, k, v, dO = (oracle_c.gen_random(cfg.n, cfg.d, 7 + i) for i in range(4))
    a = oracle_c.run(cfg, q, k, v, dO)
    b = r64.run(cfg, q, k, v, dO)
    assert np.array_equal(a.tables, b.tables)
    for key in ("out", "dq", "dk", "dv"):
        assert rel_err(getattr(a, key), getattr(b, key))["max_rel"] < 1e-4, key

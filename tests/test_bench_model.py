"""bench.py's work model (CPU): the per-stage algorithmic bytes and FLOPs the
bench line's roofline fractions divide by, checked against SURVEY.md §8(d)'s
per-unit formulas written out by hand for C3 (N = 65536, d = 64, B = 16,
K = 8, L = 3, L_e = 3, 16 units)."""
import bench

N, D, B, K, L, UNITS = 65536, 64, 16, 8, 3, 16


def test_c3_fine_kv_bytes_and_flops_follow_the_survey():
    w = bench.algorithmic_work(N, L, UNITS)
    # fine dK/dV: read Q, K, V, dO (bf16) + LSE, D; write dK, dV (bf16)
    assert w["bwd_kv_fine"]["bytes"] == UNITS * (12 * N * D + 8 * N) == 813694976
    # 8·d·P_fine with P_fine = N·K·B (query, key) pairs
    assert w["bwd_kv_fine"]["flops"] == UNITS * 8 * D * N * K * B == 68719476736


def test_c3_pairs_and_whole_path_totals():
    w = bench.algorithmic_work(N, L, UNITS)
    # E = K·L_e (fine + two coarse levels) + the coarsest level's blocks = 25
    assert w["E"] == 25
    assert w["pairs"] == UNITS * N * 25 * B
    assert w["fwd_total"]["flops"] == UNITS * 4 * D * N * 25 * B
    assert w["bwd_total"]["bytes"] == UNITS * (16 * N * D + 8 * N)


def test_stage_roofline_fraction_is_work_over_time_over_peak():
    w = bench.algorithmic_work(N, L, UNITS)
    peaks = {"bf16_tflops": 1700.6, "hbm_gbs": 6451.8}
    kv = bench.stage_roofline("bwd_kv_fine", 0.4842, w, peaks)
    gbs = w["bwd_kv_fine"]["bytes"] / 0.4842e-3 / 1e9
    assert kv["gbs"] == round(gbs, 1)
    assert kv["hbm_frac"] == round(gbs / 6451.8, 4)
    assert kv["tensor_frac"] == round(w["bwd_kv_fine"]["flops"] / 0.4842e-3 / 1e12 / 1700.6, 4)
    # its bytes reach the HBM roof before its FLOPs reach the tensor roof
    assert kv["bound"] == "hbm" and 0.2 < kv["hbm_frac"] < 0.3

"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libllsa_ref32.so, compiled
from /root/reference/proj/src by oracle/Makefile) in THIS container and stores
its outputs as small fixtures, because /root/reference does not exist on the
GPU box.  Usage:  make -C oracle && python tests/golden/make_golden.py

Fixtures
  kats.json            hand-worked known-answer tests transcribed from the
                       reference's own unit tests (file:line cited per entry)
  ref_small.npz        full path (pyramids, tables, plan, forward, CSC,
                       gradients) on tiny configs, both reweight modes
  ref_tables.npz       selection tables + CSC at the BASELINE configs
                       (N = 4096 … 65536, d = 64, bf16-rounded inputs)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Config, Reference, bf16_round  # noqa: E402

# (name, config, seed, bf16 inputs)
SMALL = [
    ("n256_scalekv", Config(256, 8, 4, 2, 2, 2), 23, False),
    ("n256_logitbias", Config(256, 8, 4, 2, 2, 2, reweight_mode=1), 23, False),
    ("n128_noenrich", Config(128, 8, 4, 2, 2, 0), 17, False),
    ("n128_partial", Config(128, 8, 4, 2, 2, 1), 29, False),
    ("n64_dense", Config(64, 8, 4, 16, 1, 0), 7, False),
    ("n256_unsafe", Config(256, 8, 4, 2, 2, 2, safe_softmax=False), 37, False),
    ("n1024_d64_b16", Config(1024, 64, 16, 4, 1, 1), 42, True),
]

TABLES = [
    ("c1_n4096_L1", Config(4096, 64, 16, 8, 1, 1), 42),
    ("c1_n4096_L2", Config(4096, 64, 16, 8, 2, 2), 42),
    ("c2_n16384_L2", Config(16384, 64, 16, 8, 2, 2), 42),
    ("c3_n65536_L3", Config(65536, 64, 16, 8, 3, 3), 42),
    ("c3p_n65536_L2", Config(65536, 64, 16, 8, 2, 2), 42),
]


def inputs(ref: Reference, cfg: Config, seed: int, bf16: bool):
    arrs = [ref.gen_random(cfg.n, cfg.d, seed + i) for i in range(4)]
    return [bf16_round(a) for a in arrs] if bf16 else arrs


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kats() -> dict:
    """Known answers transcribed from the reference's unit tests."""
    return {
        "max_levels": {  # P/tests/test_core.cpp:30-39
            "cases": [[65536, 16, 3], [65535, 16, 2], [16384, 16, 2], [256, 4, 3],
                      [16, 4, 1], [8, 4, 0], [4, 2, 1], [1, 2, 0]]},
        "effective_block_count": {  # P/tests/test_core.cpp:111-127, acceptance A8
            "cases": [[[16384, 64, 16, 8, 2, 2], 20], [[16384, 64, 16, 8, 2, 1], 16],
                      [[16384, 64, 16, 8, 2, 0], 8], [[256, 16, 4, 2, 2, 2], 8],
                      [[64, 4, 4, 2, 1, 1], 6]]},
        "validate": {  # P/tests/test_core.cpp:67-109 ([n,d,B,K,L,Le], status)
            "cases": [[[0, 4, 4, 1, 1, 0], 1], [[64, 0, 4, 1, 1, 0], 1],
                      [[64, 4, 1, 1, 1, 0], 1], [[64, 4, 0, 1, 1, 0], 1],
                      [[1 << 33, 4, 16, 2, 1, 0], 1], [[64, 4, 4, 1, 0, 0], 3],
                      [[64, 4, 4, 1, 3, 0], 3], [[64, 4, 4, 1, 2, 3], 3],
                      [[64, 4, 4, 1, 2, 2], 0], [[100, 4, 3, 1, 2, 0], 2],
                      [[99, 4, 3, 1, 2, 0], 0], [[4096, 4, 16, 16, 2, 0], 0],
                      [[4096, 4, 16, 17, 2, 0], 4], [[4096, 4, 16, 0, 2, 0], 4],
                      [[256, 4, 4, 64, 1, 0], 0], [[256, 4, 4, 65, 1, 0], 4]]},
        "pyramid": [  # P/tests/test_pyramid.cpp:23-48 (column, B, L, level, expected)
            {"x": [1, 3, 5, 7], "B": 2, "L": 1, "level": 1, "expect": [2, 6]},
            {"x": [0, 1, 2, 3, 4, 5, 6, 7], "B": 4, "L": 1, "level": 1,
             "expect": [1.5, 5.5]},
            {"x": list(range(16)), "B": 2, "L": 2, "level": 2,
             "expect": [1.5, 5.5, 9.5, 13.5]}],
        "pool_backward": [  # P/tests/test_pyramid.cpp:95-111
            {"g": [6], "B": 2, "hops": 1, "expect": [3, 3]},
            {"g": [4], "B": 2, "hops": 2, "expect": [1, 1, 1, 1]}],
        "transpose": [  # P/tests/test_indexmap.cpp:94-116
            {"rows": 4, "k": 1, "idx": [1, 0, 1, 3], "key_blocks": 4,
             "offsets": [0, 1, 3, 3, 4], "flat": [1, 0, 2, 3]},
            {"rows": 5, "k": 1, "idx": [0, 1, 2, 3, 4], "key_blocks": 5,
             "offsets": [0, 1, 2, 3, 4, 5], "flat": [0, 1, 2, 3, 4]},
            {"rows": 2, "k": 2, "idx": [0, 1, 0, 1], "key_blocks": 2,
             "offsets": [0, 2, 4], "flat": [0, 1, 0, 1]}],
        "dump_selection": {  # P/tests/test_selection.cpp:296-307
            "tables": [[0, 3], [1, 2]],
            "text": "level 0 / row 0: 0 3\nlevel 0 / row 1: 1 2\n"},
        "ties": {  # P/tests/test_selection.cpp:93-105: equal keys → first K ids
            "key_rows": 10, "d": 3, "key_row": [1, 2, 3], "q_rows": 4, "q_seed": 77,
            "top_k": 4, "expect_row": [0, 1, 2, 3]},
    }


def main() -> None:
    ref = Reference(32)
    ref.set_threads(0)
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats(), f, indent=1)

    small = {}
    for name, cfg, seed, bf in SMALL:
        q, k, v, dO = inputs(ref, cfg, seed, bf)
        r = ref.run(cfg, q, k, v, dO)
        small[f"{name}/cfg"] = np.array([cfg.n, cfg.d, cfg.block_size, cfg.top_k,
                                         cfg.levels, cfg.enrich_levels,
                                         cfg.reweight_mode, int(cfg.safe_softmax),
                                         seed, int(bf)], np.int64)
        for key in ("pyr_q", "pyr_k", "pyr_v", "tables", "out", "row_max",
                    "row_denom", "csc_offsets", "csc_flat", "dq", "dk", "dv",
                    "plan_level", "plan_block", "plan_weight"):
            small[f"{name}/{key}"] = getattr(r, key)
        small[f"{name}/checksum"] = np.array([r.checksum], np.uint64)
        small[f"{name}/macs"] = np.array([r.macs], np.uint64)
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **small)

    tabs = {}
    for name, cfg, seed in TABLES:
        q, k, v, dO = inputs(ref, cfg, seed, True)
        want_bwd = cfg.n <= 16384
        r = ref.run(cfg, q, k, v, dO if want_bwd else None)
        tabs[f"{name}/cfg"] = np.array([cfg.n, cfg.d, cfg.block_size, cfg.top_k,
                                        cfg.levels, cfg.enrich_levels, seed], np.int64)
        tabs[f"{name}/tables"] = r.tables
        tabs[f"{name}/out_sha256"] = np.array([sha(r.out)])
        tabs[f"{name}/pyr_k_sha256"] = np.array([sha(r.pyr_k)])
        if want_bwd:
            tabs[f"{name}/csc_offsets"] = r.csc_offsets
            tabs[f"{name}/csc_flat"] = r.csc_flat
        print(name, "tables", r.tables.shape, "stage ms", [round(s, 1) for s in r.stage_ms])
    np.savez_compressed(os.path.join(HERE, "ref_tables.npz"), **tabs)


if __name__ == "__main__":
    main()

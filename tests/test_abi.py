"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/llsa_cuda.h declares, and its host-only entry points
(config validation, sizes, analytic work counters) agree with the oracle and
the reference's known answers.  No kernel is launched here."""
import ctypes as C

import pytest

import paper_2512_16615_b200 as llsa
from paper_2512_16615_b200 import _lib
from oracle import Config


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == declared
    assert lib.llsa_abi_version() == 1


def test_shim_library_exports_reference_api():
    import os
    import subprocess
    so = os.path.join(os.path.dirname(_lib.LIB_PATH), "libllsa.so")
    if not os.path.exists(so):
        pytest.skip("C++ shim not built")
    syms = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True,
                          text=True).stdout
    for fn in ("llsa::build_pyramid", "llsa::pool_backward", "llsa::select_coarsest",
               "llsa::select_level", "llsa::hierarchical_topk", "llsa::transpose_indices",
               "llsa::transpose_all", "llsa::build_plan", "llsa::llsa_forward",
               "llsa::llsa_backward", "llsa::kv_backward", "llsa::validate_config",
               "llsa::max_levels", "llsa::effective_block_count", "llsa::input_checksum",
               "llsa::dump_selection"):
        assert fn + "(" in syms, fn


def test_status_names_cover_reference_errors():
    lib = _lib.load()
    names = [lib.llsa_status_name(i).decode() for i in range(1, 14)]
    assert names == ["ConfigError", "DivisibilityError", "LevelError", "TopKError",
                     "ShapeMismatch", "IndexOutOfRange", "NonFiniteError", "StaleState",
                     "FormatError", "IoError", "PrecisionError", "NotSquareBlock",
                     "OracleCapExceeded"]


def test_max_levels_kats(golden):
    for n, b, want in golden["kats"]["max_levels"]["cases"]:
        assert llsa.max_levels(n, b) == want


def test_validate_matches_kats_and_oracle(golden, oracle_c):
    for (n, d, b, k, L, le), want in golden["kats"]["validate"]["cases"]:
        cfg = llsa.LLSAConfig(n, d, b, k, L, le)
        if want == 0:
            llsa.validate_config(cfg)
        else:
            with pytest.raises(llsa.Error) as e:
                llsa.validate_config(cfg)
            assert type(e.value).code == want
        assert oracle_c.validate(Config(n, d, b, k, L, le))[0] == want
    for (n, d, b, k, L, le), want in golden["kats"]["effective_block_count"]["cases"]:
        assert llsa.validate_config(llsa.LLSAConfig(n, d, b, k, L, le)).effective_blocks == want
    assert llsa.validate_config(llsa.LLSAConfig(64, 16, 4, 2, 1, 0)).scale == 0.25
    with pytest.raises(llsa.ConfigError):
        llsa.validate_config(llsa.LLSAConfig(64, 4, 4, 1, 1, 0, softmax_scale=-1.0))


def test_validation_is_total():
    # P/tests/test_core.cpp:129-159: every config validates or raises one typed error
    seen = 0
    for n in (0, 1, 4, 63, 64, 100, 4096):
        for d in (0, 1, 16):
            for b in (0, 1, 2, 4, 16):
                for k in (0, 1, 2, 64):
                    for L in (0, 1, 2, 5):
                        for le in (0, 1, 2, 6):
                            try:
                                llsa.validate_config(llsa.LLSAConfig(n, d, b, k, L, le))
                            except (llsa.ConfigError, llsa.LevelError, llsa.DivisibilityError,
                                    llsa.TopKError):
                                pass
                            seen += 1
    assert seen == 7 * 3 * 5 * 4 * 4 * 4


@pytest.mark.parametrize("cfg", [Config(256, 8, 4, 2, 2, 2), Config(16384, 64, 16, 8, 2, 2),
                                 Config(65536, 64, 16, 8, 3, 3), Config(4096, 64, 16, 8, 1, 1),
                                 Config(128, 8, 4, 2, 2, 0)])
def test_sizes_and_analytic_counters(cfg):
    lib = _lib.load()
    c = llsa.LLSAConfig(cfg.n, cfg.d, cfg.block_size, cfg.top_k, cfg.levels,
                        cfg.enrich_levels).c()
    assert lib.llsa_pyramid_rows(cfg.n, cfg.block_size, cfg.levels) == cfg.pyramid_rows()
    assert lib.llsa_table_entries(C.byref(c)) == sum(cfg.table_rows()) * cfg.top_k
    # selection.cpp:75-77,145-147
    top = cfg.level_tokens(cfg.levels)
    sel = top * top * cfg.d + sum(cfg.level_tokens(l) * cfg.top_k * cfg.block_size * cfg.d
                                  for l in range(1, cfg.levels))
    assert lib.llsa_select_mul_accs(C.byref(c)) == sel
    assert lib.llsa_forward_mul_accs(C.byref(c)) == (cfg.n * cfg.effective_blocks *
                                                     cfg.block_size * cfg.d)


def test_backward_counter_matches_reference_fixture(golden):
    g = golden["small"]
    for name in ("n256_scalekv", "n128_noenrich", "n128_partial"):
        n, d, b, k, L, le = (int(x) for x in g[f"{name}/cfg"][:6])
        c = llsa.LLSAConfig(n, d, b, k, L, le).c()
        lib = _lib.load()
        total = (lib.llsa_select_mul_accs(C.byref(c)) + lib.llsa_forward_mul_accs(C.byref(c)) +
                 lib.llsa_backward_mul_accs(C.byref(c)))
        assert total == int(g[f"{name}/macs"][0]), name

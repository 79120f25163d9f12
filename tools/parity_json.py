"""Dev: turns the GPU parity log (LLSA_PARITY_LOG=gpurun_out/parity.jsonl,
written by tests/test_gpu_parity.py::test_full_size_tensor_core_path_matches_reference)
into profiles/r2_parity.json (the table DESIGN.md's precision section cites).
Usage: python tools/parity_json.py gpurun_out/parity.jsonl profiles/r2_parity.json"""
import json
import sys

src, dst = sys.argv[1], sys.argv[2]
cases = [json.loads(line) for line in open(src) if line.strip()]
doc = {
    "what": "tcgen05 handle path vs the compiled unmodified reference "
            "(oracle/_ref/libllsa_ref32.so, f32 build) on bf16-rounded reference gen_random "
            "inputs, 1 unit per case; tests/test_gpu_parity.py::"
            "test_full_size_tensor_core_path_matches_reference (default, unordered coarse "
            "reductions)",
    "bars": {"tables": "bit-exact", "max_rel": 0.02, "fro": 0.01, "p99_row": 0.06,
             "lse_max_abs": 0.01},
    "metrics": "max_rel = max|d|/max|ref|; fro = ||d||/||ref||; p99_row / worst_row over rows "
               "with ||ref_row|| >= 1e-3 max row norm",
    "cases": cases,
}
json.dump(doc, open(dst, "w"), indent=1)
print(f"{len(cases)} cases -> {dst}")

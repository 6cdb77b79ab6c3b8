"""CPU checks of the report writer."""
import numpy as np

from paper_2011_12875_b200 import report


def test_checksum_matches_reference_fnv1a(port):
    # acceptance gate (tests/acceptance.cpp:249-275) on the bitwise oracle
    q = port.synthetic(64, 14, 8, seed=600)
    assert report.checksum_hex(port.run(q, want=("forces",))["forces"]) == "dd6d6cc7a1c2e358"


def test_csv_columns_follow_reference_header():
    row = {"variant": "gpu-b200", "natoms": 2000, "nnbor": 26, "twojmax": 8, "steps": 10,
           "wall_ms_per_step": 0.158, "katom_steps_per_s": 12658.2, "speedup_vs_baseline": 240.0,
           "peak_bytes_total": 123, "force_checksum": "0123456789abcdef",
           "step_tflops": 13.6, "fp64_peak_frac": 0.365}
    lines = report.write_report_csv([row]).splitlines()
    assert lines[0] == report.CSV_HEADER + ",step_tflops,fp64_peak_frac"
    assert lines[1].split(",")[:5] == ["gpu-b200", "2000", "26", "8", "10"]
    assert lines[1].split(",")[9] == "0123456789abcdef"
    assert report.checksum_hex(np.zeros(0)) == "cbf29ce484222325"

"""CLI `simulate` (tools/ilsim_main.cpp:126-186) report formats and errors."""
import subprocess
import sys

import numpy as np
import pytest

from paper_2105_05821_b200.cli import phase_cpi, phase_cpi_csv, sim_report_csv

GOLD = __import__("conftest").GOLDEN
ROOT = GOLD.parents[1]


def test_phase_cpi_windows():  # metrics.cpp:18-31
    cpi, partial = phase_cpi(np.array([1, 2, 3, 4, 5]), 2)
    assert cpi == [1.5, 3.5, 5.0] and partial
    assert phase_cpi_csv(cpi) == "window_index,cpi\n0,1.5\n1,3.5\n2,5\n"


def test_sim_report_csv_format():  # metrics.cpp:33-40
    r = {"instructions": 3, "total_cycles": 9, "cpi": 3.0, "sum_fetch": 6, "delta": 3, "drain_cycles": 3,
         "overflow_stall_cycles": 0, "empty": False}
    assert sim_report_csv(r).splitlines()[1] == "3,9,3,6,3,3,0,0"


def test_cli_errors_like_reference(tmp_path):
    out = subprocess.run([sys.executable, "-m", "paper_2105_05821_b200", "simulate", "--trace",
                          str(tmp_path / "missing.trace"), "--oracle", "--report", str(tmp_path / "r.csv")],
                         capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 1 and out.stderr.startswith("error: ")


@pytest.mark.gpu
def test_cli_simulate_matches_port(tmp_path, port):
    rep = tmp_path / "r.csv"
    out = subprocess.run([sys.executable, "-m", "paper_2105_05821_b200", "simulate", "--trace",
                          str(GOLD / "mix_3000_s4.trace"), "--oracle", "--parallel", "5", "--report", str(rep),
                          "--throughput", str(tmp_path / "t.csv")], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    from paper_2105_05821_b200.formats import read_trace
    want = port.simulate(read_trace(GOLD / "mix_3000_s4.trace"), oracle=True, k=5)
    row = rep.read_text().splitlines()[1].split(",")
    assert int(row[1]) == want["total_cycles"]
    phase = (tmp_path / "r.csv.phase.csv").read_text().splitlines()
    assert phase[0] == "window_index,cpi" and len(phase) == 101
    assert out.stdout.startswith("simulated 3000 instructions: ")

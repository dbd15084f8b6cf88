"""Bench record formats and the `bcad_bench` CLI (include/bcad/bench.hpp,
SURVEY §8(f) row 4). CPU part: record emission / parsing and CLI config
errors need no device (tests/cpp/cpu_bench_records.cpp). GPU part: a tiny
end-to-end CLI run whose CSV rows carry the device implementation names."""
import csv
import io
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPU_PROG = os.path.join(ROOT, "tests", "cpp", "bin", "cpu_bench_records")
CLI = os.path.join(ROOT, "paper_1810_08297_b200", "bin", "bcad_bench")
HEADER = ("workload,impl,n,arity,reps,min_ns,median_ns,mean_ns,tape_nodes,peak_cached_bytes,"
          "transcendental_evals,rng_seed")


def test_record_formats_and_cli_errors_cpu():
    r = subprocess.run([CPU_PROG], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


@pytest.mark.parametrize("args,code", [(["--help"], 0), ([], 1), (["hmlstm", "--n", "0"], 1),
                                       (["hmlstm", "--impl", "alien"], 1), (["arity", "--arities", "33"], 1),
                                       (["hmlstm", "--precision", "f16"], 1)])
def test_cli_exit_codes_cpu(args, code):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=60)
    assert r.returncode == code, r.stderr


@pytest.mark.gpu
def test_cli_tiny_run_gpu():
    r = subprocess.run([CLI, "hmlstm", "--n", "8,16", "--reps", "2", "--warmup", "1", "--precision", "f32"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == HEADER
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 8
    assert {row["impl"] for row in rows} == {"forward-only", "mixed-cache", "mixed-recompute", "reverse-unfused"}
    for row in rows:
        assert int(row["min_ns"]) > 0 and int(row["min_ns"]) <= int(row["median_ns"])
        if row["impl"] == "reverse-unfused":
            n = int(row["n"])
            assert int(row["transcendental_evals"]) == 3 * n * n
            assert int(row["tape_nodes"]) == 14

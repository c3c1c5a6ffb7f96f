"""GPU: tools/sigbench emits the reference's CSV schema (bench.cpp:192-229,
tests/test_bench.cpp:126-141) with B200 timings, including the paper grid."""
import csv
import io
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tools", "sigbench")
HEADER = "kernel,batch,seq_len,dim,depth,dtype,reps,mean_ms,std_ms,min_ms,counter"


def run(*args):
    r = subprocess.run([EXE, *args], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_csv_grid_shape_and_values():
    out = run("--batch-sizes", "4,8", "--seq-lens", "50", "--dims", "2,3", "--depths", "3", "--repeats", "3",
              "--warmup", "1", "--dtype", "f32")
    lines = out.strip().splitlines()
    assert lines[0] == HEADER
    rows = list(csv.DictReader(io.StringIO(out)))
    assert len(rows) == 2 * 2 * 2  # points x kernels
    for r in rows:
        assert r["dtype"] == "f32" and r["reps"] == "3"
        assert float(r["min_ms"]) > 0 and float(r["mean_ms"]) >= float(r["min_ms"])
        # the reference's structural counter (bench.cpp:37-48): L-1 folds / depth scan passes
        assert int(r["counter"]) == (int(r["seq_len"]) - 1 if r["kernel"] == "sequential" else int(r["depth"]))


def test_paper_grid_markdown():
    out = run("--paper-grid", "--dims", "3", "--kernels", "sequential", "--repeats", "2", "--warmup", "1",
              "--format", "markdown")
    lines = out.strip().splitlines()
    assert lines[0].startswith("| kernel |") and len(lines) == 2 + 15

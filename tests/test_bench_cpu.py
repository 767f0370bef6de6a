"""CPU checks of bench.py's host logic: workload parsing and the reference (oracle) arm."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse_workload():
    assert bench.parse_workload("28,3,lex") == (28, 3, "lex", {})
    n, d, o, ex = bench.parse_workload("24,8,lex,so,cw=12")
    assert (n, d, o) == (24, 8, "lex") and ex == {"self_orthogonal": True, "constant_weight": 12}
    b = bench.parse_workload("12,3,lex,basis=seed:4")[3]["basis"]
    assert len(b) == 12 and len(set(b)) == 12
    assert bench.parse_workload("5,2,lex,basis=gray")[3]["basis"] == [1, 3, 6, 12, 24]


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--ref-log2", "12"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "checks/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_b200_arm_source_compiles():
    import py_compile
    py_compile.compile(os.path.join(ROOT, "bench.py"), doraise=True)

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
    # a small bench workload with a golden row: the oracle arm runs the WHOLE workload per step
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
                          "--workload", "24,3,lex"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "checks/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["M"] == 524288 and line["config"]["w_def"] == bench.golden_row("24,3,lex")["w_def"]
    assert line["cpu_baseline"]["host_threads"] >= 1


def test_cpu_baseline_fields():
    cb = bench.cpu_baseline(12, 3, "lex", {}, 10 ** 6, budget_s=1.0)
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] > 0
    assert cb["o1_threads"]["cores"] == cb["host_threads"] and cb["o1_1thread"]["value"] > 0


def test_golden_row_lookup():
    assert bench.golden_row("28,3,lex")["M"] == 8388608
    assert bench.golden_row("28,3,lex,so") is None


def test_b200_arm_source_compiles():
    import py_compile
    py_compile.compile(os.path.join(ROOT, "bench.py"), doraise=True)

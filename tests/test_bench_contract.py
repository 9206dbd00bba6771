"""bench.py's JSON contract, checked on CPU through the reference arm (oracle/_ref on the host
cores; the GPU arm's line is produced on the B200 and committed under profiles/)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REQUIRED = {"metric": str, "value": (int, float), "unit": str, "n_gpus": int, "steps": int, "warmup": int,
            "ms_per_step": (int, float), "higher_is_better": bool, "scaling": str, "dtype": str, "data": str,
            "config": dict}


def test_reference_arm_line_on_cpu():
    from oracle import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k, t in REQUIRED.items():
        assert isinstance(d[k], t), (k, d.get(k))
    assert d["warmup"] >= 3                       # timing rule: W >= 3
    assert d["config"]["workload"] == "c1"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_committed_gpu_line_has_contract_keys():
    """The committed B200 line (profiles/r01_bench_c2.json) carries the contract's keys."""
    d = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_c2.json")))
    for k, t in REQUIRED.items():
        assert isinstance(d[k], t), k
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_mhz"] and d["config"]["workload"] == "c2"


def test_reference_arm_never_loads_the_product_library():
    """The reference arm (and the CPU edge generators it uses) runs the unmodified reference
    only: after a full --impl reference run the process has mapped oracle/_ref and the
    oracle restatement, never paper_2112_01743_b200/lib/libchebpr_b200.so."""
    from oracle import REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', '--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('PRODUCT' if 'libchebpr_b200' in maps else 'CLEAN', 'REF' if 'libchebpr_ref' in maps else 'NOREF')\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip().splitlines()[-1] == "CLEAN REF"

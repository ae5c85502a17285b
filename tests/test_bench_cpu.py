"""bench.py's CPU-only arm (--impl reference: the oracle on the host cores) runs and prints the
contract's JSON line; it needs no GPU, so it is checked here (`-m "not gpu"`)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_contract_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--net", "tiny", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    d = json.loads(res.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["dtype"] == "u32" and d["steps"] == 1
    assert "whole network once" in d["cpu_baseline"]["sample"]  # measured, not extrapolated


def test_reference_arm_imports_no_product_code():
    """The reference arm is the oracle alone: running it must not load the product library or
    import the product package (its planner came from libsecn)."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--net', 'tiny', '--steps', '2', "
            "'--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nfinally:\n"
            "    bad = [m for m in sys.modules if m.startswith('paper_2506_11586_b200')]\n"
            "    maps = open('/proc/self/maps').read()\n"
            "    assert not bad and 'libsecn' not in maps, (bad, 'libsecn' in maps)\n"
            "    print('NOPRODUCT')")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "NOPRODUCT" in res.stdout


def test_oracle_chunks_cover_network_once():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)

    class O:
        def __init__(self, M, S):
            self.M, self.S = M, S

    states = [{"opl": O(3, 2)}, {"opl": O(1, 1)}, {"opl": O(10, 1)}, {"opl": O(5, 3)}]
    for parts in (1, 2, 3, 7, 40):
        chunks, total = bench.oracle_chunks(states, parts)
        assert total == 6 + 1 + 10 + 15 and len(chunks) == parts
        seen = {i: [] for i in range(4)}
        for rs in chunks:
            for li, lo, hi in rs:
                assert lo < hi
                seen[li].extend(range(lo, hi))
        for li, st in enumerate(states):
            assert seen[li] == list(range(st["opl"].M * st["opl"].S))
    chunks, total = bench.oracle_chunks(states, 1, frac=0.1)
    assert [(li, lo, hi) for li, lo, hi in chunks[0]] == [(0, 0, 1), (1, 0, 1), (2, 0, 1), (3, 0, 2)]

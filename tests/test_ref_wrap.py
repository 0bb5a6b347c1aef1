"""The reference's OWN test files, compiled unmodified (Makefile target
`refwrap`, outputs in oracle/_ref/wrap), with the k-hop path on the B200:
k_hop_count / k_hop_frontier replaced at link time (ld --wrap) and the Cypher
VarLenTraverse step bound to mgk_walk_targets.

* proj/tests/test_execute.cpp + test_bench.cpp (doctest-compatible shim):
  every case must pass with the k-hop calls answered by the GPU;
* proj/tests/acceptance/acceptance_main.cpp: criterion c1 (20 RMAT graphs x
  50 seeds x k=1,2,3,6 x 2 modes = 8,000 k_hop_count calls vs BfsOracle);
* [*min..max] walks in both directions through the reference's parse ->
  plan -> execute, against the reference-generated walk_pins.json.
"""
import json
import re
import subprocess
from pathlib import Path

import pytest

from conftest import load_golden

ROOT = Path(__file__).resolve().parents[1]
RW = ROOT / "oracle" / "_ref" / "wrap"
need = pytest.mark.skipif(not (RW / "ref_tests_gpu").exists(), reason="refwrap binaries not built (needs /root/reference)")


def routed(stderr: str) -> dict:
    m = re.search(r"routed to the GPU: k_hop_count (\d+), k_hop_frontier (\d+), walks (\d+)", stderr)
    assert m, stderr[-2000:]
    return {"count": int(m.group(1)), "frontier": int(m.group(2)), "walks": int(m.group(3))}


@need
def test_wrapped_symbols_and_host_cases():
    """CPU: the binaries carry the --wrap replacements, and the reference's
    host-only cases (generator, statistics, schedules, reports, edge lists)
    pass unchanged."""
    syms = subprocess.run(["nm", str(RW / "ref_tests_gpu")], capture_output=True, text=True).stdout
    assert "__wrap__ZN8matgraph11k_hop_countERKNS_13PropertyGraphERKNS_9KHopQueryE" in syms
    assert "__wrap__ZN8matgraph14k_hop_frontierERKNS_13PropertyGraphERKNS_9KHopQueryE" in syms
    r = subprocess.run([str(RW / "ref_tests_gpu"), "-tc=rmat*,the top-left*,summary*,schedules*,reports*,"
                        "report files*,edge lists*,seed picking*,the oracle validates*"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "| 0 failed" in r.stdout


@need
@pytest.mark.gpu
def test_reference_unit_tests_on_gpu():
    r = subprocess.run([str(RW / "ref_tests_gpu")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    n = routed(r.stderr)
    # test_execute.cpp:104-173 and test_bench.cpp:115-138, 262-317 reach the GPU
    assert n["count"] > 100 and n["frontier"] >= 1 and n["walks"] > 0, n


@need
@pytest.mark.gpu
def test_reference_acceptance_c1_on_gpu():
    r = subprocess.run([str(RW / "acceptance_gpu")], capture_output=True, text=True, timeout=900)
    c1 = [ln for ln in r.stdout.splitlines() if " c1: " in ln]
    assert c1 and c1[0].startswith("PASS c1: 8000/8000"), r.stdout[-3000:]
    assert routed(r.stderr)["count"] >= 8000


@need
@pytest.mark.gpu
def test_reference_cypher_varlen_walks_on_gpu():
    w = load_golden("walk_pins")
    want = {}
    for g in w["graphs"]:
        for c in g["cases"]:
            key = (f"s{g['scale']}r{g['rng_seed']}", c["seed"], c["min"], c["max"])
            want[key + ("out",)] = c["ids"]
            want[key + ("in",)] = c["in_ids"]
    for c in w["cycle_loop"]["cases"]:
        key = ("cycle_loop", c["seed"], c["min"], c["max"])
        want[key + ("out",)] = c["ids"]
        want[key + ("in",)] = c["in_ids"]
    r = subprocess.run([str(RW / "varlen_gpu")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    got = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(got) == len(want)
    for q in got:
        key = (q["graph"], q["seed"], q["min"], q["max"], q["dir"])
        assert q["ids"] == want[key], key
    assert routed(r.stderr)["walks"] >= len(want)

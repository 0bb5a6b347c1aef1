"""Runs the C++ drop-in's own test program (tests/cpp/test_dropin.cpp):
`--cpu` cases here, every case (incl. acceptance c1) on the GPU box."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "build" / "test_dropin"


def ensure_built():
    if not EXE.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT), "cpptest"], check=True)


def test_cpp_dropin_host_cases():
    ensure_built()
    r = subprocess.run([str(EXE), "--cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout


def test_dropin_exports_reference_signatures():
    """The drop-in library defines the reference's k-hop entry points (mangled
    C++ names of namespace matgraph, execute.hpp:65-68, bench.hpp:62-68)."""
    ensure_built()
    out = subprocess.run(["nm", "-DC", str(ROOT / "paper_1905_01294_b200" / "lib" / "libmatgraph_b200.so")],
                         capture_output=True, text=True).stdout
    for sym in ("matgraph::k_hop_count(matgraph::PropertyGraph const&, matgraph::KHopQuery const&)",
                "matgraph::k_hop_frontier(matgraph::PropertyGraph const&, matgraph::KHopQuery const&)",
                "matgraph::build_bench_graph(",
                "matgraph::pick_seeds(matgraph::PropertyGraph const&, unsigned long, unsigned long)",
                "matgraph::run_khop_benchmark("):
        assert sym in out, sym


@pytest.mark.gpu
def test_cpp_dropin_all_cases():
    ensure_built()
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout

"""Harness pieces (bench.cpp mirrors) pinned by proj/tests/test_bench.cpp."""
import pytest

from paper_1905_01294_b200 import harness as H
from paper_1905_01294_b200.khop import ContractError


def test_summary_statistics():  # test_bench.cpp:148-168
    runs = [H.SeedRun(0, 2, 10), H.SeedRun(1, 4, 30), H.SeedRun(2, 6, 20), H.SeedRun(3, 8, 40)]
    s = H.summarize(runs)
    assert (s.mean_us, s.median_us, s.p99_us, s.mean_count) == (25.0, 25.0, 40.0, 5.0)
    odd = H.summarize([H.SeedRun(0, 0, 1), H.SeedRun(1, 0, 100), H.SeedRun(2, 0, 2)])
    assert odd.median_us == 2.0
    with pytest.raises(ContractError, match="cannot summarize an empty run list"):
        H.summarize([])


def test_schedule_validation():  # test_bench.cpp:170-188
    s = H.BenchSchedule([1, 2], [10])
    with pytest.raises(ContractError, match="schedule pairs 2 hop counts with 1 seed counts"):
        s.validate()
    with pytest.raises(ContractError, match="seed count for k=2 must be at least 1"):
        H.BenchSchedule([1, 2], [10, 0]).validate()
    with pytest.raises(ContractError, match=r"hop count 0 outside \[1, 32\]"):
        H.BenchSchedule([0, 2], [10, 10]).validate()
    with pytest.raises(ContractError, match=r"hop count 33 outside \[1, 32\]"):
        H.BenchSchedule([33], [1]).validate()


def test_report_csv():  # test_bench.cpp:190-209
    assert H.report_csv_string(H.KHopReport()) == (
        "k,seed,count,elapsed_us\nk,n_seeds,mean_us,median_us,p99_us,mean_count\n")
    runs = [H.SeedRun(5, 7, 10), H.SeedRun(6, 9, 20)]
    rep = H.KHopReport(sections=[H.KHopSection(2, runs, H.summarize(runs))])
    assert H.report_csv_string(rep) == ("k,seed,count,elapsed_us\n2,5,7,10\n2,6,9,20\n"
                                        "k,n_seeds,mean_us,median_us,p99_us,mean_count\n"
                                        "2,2,15,15,20,8\n")


def test_baseline_configs_shapes():
    assert H.CONFIGS["cfg2"].graph.target_unique == 67_108_864
    assert H.CONFIGS["cfg5"].seeds_per_k == (65536,) * 4
    assert H.CONFIGS["cfg1"].graph.scale == 16

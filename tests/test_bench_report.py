"""The reference's benchmark-report format (mpcdsim/bench.py), CPU part:
rank factorisation, CSV round trip, summary -- mirroring the reference's
own tests (test_bench_cli.py:20-135).  The timed cases need a GPU and live
in test_gpu_distributed.py."""

import math

import pytest

from paper_2212_11878_b200 import bench
from paper_2212_11878_b200.errors import ConfigError, MpcdError


@pytest.mark.parametrize("n,dims", [(1, (1, 1, 1)), (2, (2, 1, 1)), (4, (2, 2, 1)),
                                    (6, (3, 2, 1)), (8, (2, 2, 2)), (12, (3, 2, 2)),
                                    (16, (4, 2, 2))])
def test_rank_dims_for(n, dims):
    got = bench.rank_dims_for(n)
    assert got == dims and math.prod(got) == n


def test_rank_dims_for_rejects_nonpositive():
    with pytest.raises(ConfigError):
        bench.rank_dims_for(0)


def _recs():
    return [bench.BenchRecord(L=16, ranks=1, scheme="halo", steps=3, seconds=0.1 + 1e-17,
                              particles=40960, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=1.3e-17),
            bench.BenchRecord(L=16, ranks=2, scheme="halo", steps=3, seconds=0.07,
                              particles=40960, bytes_per_step=2.0 ** 20 / 3,
                              msgs_per_step=2.0, max_drift=2.2e-16),
            bench.BenchRecord(L=16, ranks=3, scheme="halo", steps=3, seconds=0.0, particles=0,
                              bytes_per_step=0.0, msgs_per_step=0.0, max_drift=0.0,
                              error="ConfigError: rank_dims entry 3 does not divide 16")]


def test_report_roundtrip_exact(tmp_path):
    path = tmp_path / "bench.csv"
    recs = _recs()
    bench.emit_report(recs, str(path))
    assert bench.read_report(str(path)) == recs  # repr keeps floats exact
    summary = (tmp_path / "bench.csv.summary.txt").read_text()
    assert "speedup=" in summary and "FAILED" in summary and "L=16" in summary


def test_report_refuses_empty_and_bad_header(tmp_path):
    with pytest.raises(MpcdError):
        bench.emit_report([], str(tmp_path / "x.csv"))
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(MpcdError):
        bench.read_report(str(bad))


def _golden_records():
    return [bench.BenchRecord(L=16, ranks=1, scheme="halo", steps=3, seconds=0.1 + 1e-17,
                              particles=40960, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=1.3e-17),
            bench.BenchRecord(L=16, ranks=2, scheme="halo", steps=3, seconds=0.07,
                              particles=40960, bytes_per_step=2.0 ** 20 / 3,
                              msgs_per_step=2.0, max_drift=2.2e-16),
            bench.BenchRecord(L=16, ranks=3, scheme="migration", steps=3, seconds=0.0,
                              particles=0, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=0.0, error="ConfigError: rank_dims entry 3 does not "
                              "divide 16, \"quoted\""),
            bench.BenchRecord(L=32, ranks=1, scheme="halo", steps=20, seconds=1.2345678901234,
                              particles=327680, bytes_per_step=0.0, msgs_per_step=0.0,
                              max_drift=3.5e-15),
            bench.BenchRecord(L=32, ranks=8, scheme="halo", steps=20, seconds=0.2,
                              particles=327680, bytes_per_step=123456.5, msgs_per_step=7.5,
                              max_drift=1e-300)]


def test_report_bytes_equal_reference_emit_report(tmp_path):
    """The CSV and summary files are byte-identical to the reference's
    emit_report of the same records (tests/golden/bench_report.csv, made by
    make_golden.py from the reference), and read back to the same records."""
    import os

    from conftest import GOLDEN
    path = tmp_path / "b.csv"
    bench.emit_report(_golden_records(), str(path))
    for suffix in ("", ".summary.txt"):
        with open(os.path.join(GOLDEN, "bench_report.csv" + suffix), "rb") as fh:
            assert (tmp_path / ("b.csv" + suffix)).read_bytes() == fh.read(), suffix
    assert bench.read_report(os.path.join(GOLDEN, "bench_report.csv")) == _golden_records()


def test_rank_dims_equal_reference():
    import os

    import numpy as np

    from conftest import GOLDEN
    want = np.load(os.path.join(GOLDEN, "bench_rank_dims.npy"))
    got = np.array([bench.rank_dims_for(n) for n in range(1, 65)])
    assert np.array_equal(got, want)

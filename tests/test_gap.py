import math
import warnings

import pytest

from paper_2404_03617_b200 import gap
from paper_2404_03617_b200.core import DeviceSpec

A5000 = DeviceSpec("a5000", 76.7e12, 479.375e9)


def test_reference_gap_table_pico():
    # Pico 256^2 b128 6.078 ms -> 47.2% of A5000 peak
    s = gap.MeasuredSample("pico", 0.8602e9, 128, 6.078e-3)
    eff, ach = gap.computational_efficiency(s, A5000)
    assert eff == pytest.approx(0.4723, abs=2e-3)
    assert gap.ideal_latency(0.8602e9, 128, A5000) == pytest.approx(2 * 0.8602e9 * 128 / 76.7e12)


def test_series_sorted_and_gap_width(tmp_path):
    samples = [gap.MeasuredSample("b", 2e9, 128, 0.01, 80.0), gap.MeasuredSample("a", 1e9, 128, 0.01)]
    pts = gap.gap_series(samples, A5000)
    assert [p.sample.model for p in pts] == ["a", "b"]
    assert pts[0].gap_width == pytest.approx(-math.log(pts[0].efficiency))
    path = tmp_path / "s.csv"
    gap.write_samples_csv(path, samples)
    back = gap.load_samples_csv(path)
    assert [(s.model, s.batch, s.accuracy_pct) for s in back] == [("b", 128, 80.0), ("a", 128, None)]


def test_efficiency_above_one_warns():
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        gap.computational_efficiency(gap.MeasuredSample("x", 1e12, 128, 1e-6), A5000)
    assert w


def test_bad_csv_reports_row(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("model,macs_g,batch,latency_ms,accuracy_pct\nx,notanumber,1,1,\n")
    with pytest.raises(ValueError, match="row 2"):
        gap.load_samples_csv(p)


def test_b200_device_files_and_gap_plot():
    from paper_2404_03617_b200 import gap as g

    ds, me = g.load_device("b200-datasheet"), g.load_device("b200-measured")
    assert abs(ds.op_byte - 281.25) < 1e-9 and me.peak_throughput < ds.peak_throughput
    with pytest.raises(KeyError):
        g.load_device("h100")
    pts = g.gap_series([g.MeasuredSample("pico", 0.659e9, 128, 1.1e-3, 79.9),
                        g.MeasuredSample("nx", 4.46e9, 128, 6.3e-3, None)], me)
    svg = g.gap_plot(pts, me, "gap <b200>")
    assert svg.startswith("<svg") and svg.rstrip().endswith("</svg>") and "&lt;b200&gt;" in svg
    assert svg.count("<circle") == 4

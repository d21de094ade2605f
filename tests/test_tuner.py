"""Device batch-width tuner (reference tuner.hpp:33-139; the reference's own
tests/test_tuner.cpp also runs through the C++ drop-in in test_cpp.py).

CPU: the width rule, report validation, CSV layout and argument checks.
GPU: measurements of the device SpMM kernels and a consistent report.
"""
import io

import pytest

import paper_2601_21990_b200 as bl
from paper_2601_21990_b200 import instances as I
from paper_2601_21990_b200.errors import InvalidArgument, LogicError


def test_choose_width_picks_the_minimum_and_breaks_ties_upward():
    assert bl.choose_width([bl.TuneEntry(64, 1.0, 0.5)]) == 64
    tied = [bl.TuneEntry(32, 3.0, 3.0), bl.TuneEntry(64, 1.0, 1.0), bl.TuneEntry(128, 2.0, 1.0)]
    assert bl.choose_width(tied) == 128
    with pytest.raises(InvalidArgument):
        bl.choose_width([])


def test_reports_validate_their_own_consistency():
    r = bl.TuneReport(entries=[bl.TuneEntry(32, 1.0, 1.0), bl.TuneEntry(64, 0.5, 0.25)],
                      chosen_width=64)
    r.validate()
    r.chosen_width = 32
    with pytest.raises(LogicError):
        r.validate()
    r = bl.TuneReport(entries=[bl.TuneEntry(32, -1.0, -1.0)], chosen_width=32)
    with pytest.raises(LogicError):
        r.validate()


def test_csv_layout():
    r = bl.TuneReport(entries=[bl.TuneEntry(1, 0.5, 0.5), bl.TuneEntry(2, 1e-5, 5e-6)],
                      chosen_width=2)
    out = io.StringIO()
    bl.write_tune_csv(out, r)
    assert out.getvalue() == "width,total_s,per_column_s,chosen\n1,0.5,0.5,0\n2,1e-05,5e-06,1\n"
    assert bl.default_tune_widths() == [32, 64, 128, 256, 512, 1024, 2048]


def test_bad_arguments_are_rejected_before_any_device_work():
    A = I.set_cover(10, 10, 0.2, 3).A
    with pytest.raises(InvalidArgument):
        bl.measure_spmm(A, 0, 10)
    with pytest.raises(InvalidArgument):
        bl.measure_spmm(A, 4, 2)
    with pytest.raises(InvalidArgument):
        bl.tune_batch_width(A, [], 3)


@pytest.mark.gpu
def test_width_one_total_equals_per_column():
    A = I.set_cover(40, 50, 0.1, 7).A
    total, per_column, _ = bl.measure_spmm(A, 1, 3)
    assert total == per_column
    assert total >= 0.0


@pytest.mark.gpu
def test_tuning_the_c2_matrix_gives_a_consistent_report():
    A = I.config_problem("c2").A
    widths = [32, 128, 512, 2048]
    r = bl.tune_batch_width(A, widths, 5)
    assert [e.width for e in r.entries] == widths
    assert r.chosen_width in widths
    r.validate()
    for e in r.entries:
        assert e.total_s > 0.0
        assert e.per_column_s == pytest.approx(e.total_s / e.width)
    # wider blocks amortise the matrix: 2048 columns cost less per column than 32
    per = {e.width: e.per_column_s for e in r.entries}
    assert per[2048] < per[32]
    out = io.StringIO()
    bl.write_tune_csv(out, r)
    assert out.getvalue().count("\n") == len(widths) + 1

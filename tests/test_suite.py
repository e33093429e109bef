"""Auto-tuner contract and CSV schema of the Kershaw-study driver, on the CPU with
injected runs and clocks (acceptance criterion 9, first half; bench_cli CSV round trip)."""
import os

import pytest

from paper_2110_07663_b200 import suite


class FakeClock:
    """Scripted clock: every pair of calls (start, stop) measures the next scripted duration."""

    def __init__(self, durations):
        self.d = list(durations)
        self.t = 0.0
        self.start = True

    def __call__(self):
        if not self.start:
            self.t += self.d.pop(0)
        self.start = not self.start
        return self.t


def _cands(k):
    return [suite.PreconditionerConfig("cheb_ras", (7, 3, 1), eta=i + 1) for i in range(k)]


def _run(conv=None):
    conv = conv or {}

    def run(cfg):
        return lambda: (conv.get(cfg.eta, True), 10, 1e-9)
    return run


def test_autotune_picks_injected_fastest():
    # per candidate: setup, then 3 solves; candidate 3 (eta=3) has the smallest median
    clock = FakeClock([1, 5, 5, 5,  1, 4, 4, 4,  1, 2, 9, 2,  1, 3, 3, 3])
    chosen, recs = suite.autotune(_cands(4), _run(), trials=3, timer=clock)
    assert chosen.eta == 3
    assert [r.median_s for r in recs] == [5, 4, 2, 3]


def test_autotune_tie_goes_to_list_order():
    clock = FakeClock([1, 2, 2, 2,  1, 2, 2, 2])
    chosen, _ = suite.autotune(_cands(2), _run(), trials=3, timer=clock)
    assert chosen.eta == 1


def test_autotune_never_picks_nonconverged():
    clock = FakeClock([1, 9, 9, 9,  1, 1, 1, 1])
    chosen, recs = suite.autotune(_cands(2), _run({2: False}), trials=3, timer=clock)
    assert chosen.eta == 1 and not recs[1].converged
    with pytest.raises(RuntimeError):
        suite.autotune(_cands(1), _run({1: False}), trials=1, timer=FakeClock([1, 1]))
    with pytest.raises(ValueError):
        suite.autotune([], _run())


def test_table3_space():
    names = [c.name for c in suite.table3_space(7)]
    assert names == ["Cheby-ASM(2),(7,3,1)", "Cheby-RAS(2),(7,3,1)", "Cheby-Jac(2),(7,5,3,1)", "semfem"]
    assert [c.schedule for c in suite.table3_space(9)][:3] == [(9, 5, 1), (9, 5, 1), (9, 7, 5, 1)]
    assert suite.parse_precond("cheb_jac:7,5,3,1:3", 7) == suite.PreconditionerConfig("cheb_jac", (7, 5, 3, 1), 3)


def test_csv_round_trip(tmp_path):
    rows = [suite._row(0.3, 6, 7, 79507, "Cheby-RAS(2),(7,3,1)", 12, 0.5, 0.01, 8.5e-9, True, "solve", 1)]
    path = os.path.join(tmp_path, "k.csv")
    suite.write_csv(path, rows)
    assert suite.read_csv(path) == rows
    with open(path) as f:
        assert f.readline().strip() == ",".join(suite.HEADER)

"""schedsim: the SPEC's examples and acceptance criterion 5."""

from fractions import Fraction

import pytest

from paper_2210_09147_b200 import cli, schedsim as ss


def _sim(kind, D, n=8, m=4):
    return ss.simulate(ss.SchedulePolicy(kind, D, n, m))


def test_partime_rule_example():
    ev, _ = _sim("partime", 3, 8)
    at = {(e.slot, e.stage, e.op): e.sample for e in ev}
    assert at[(6, 1, "F")] == 6 and at[(6, 1, "B")] == 2


@pytest.mark.parametrize("D", range(1, 17))
def test_partime_invariants(D):
    _, r = _sim("partime", D, 2 * D + 4)
    assert r.staleness == [2 * (D - h) for h in range(1, D + 1)]
    assert r.throughput == 1 and all(f == 0 for f in r.idle_fraction)


def test_gpipe_idle_and_throughput():
    _, r = _sim("gpipe", 4, 16, 4)
    assert all(f == Fraction(3, 7) for f in r.idle_fraction)
    for m in (1, 2, 8, 32):
        assert _sim("gpipe", 4, 2 * m, m)[1].throughput < 1


@pytest.mark.parametrize("D", [2, 3, 4, 6])
def test_pipedream_and_2bw_memory(D):
    _, r = _sim("pipedream", D, 4 * D, D)
    assert r.weight_versions == [D - s + 1 for s in range(1, D + 1)]
    assert r.staleness[-1] == 0
    _, r2 = _sim("pipedream2bw", D, 4 * D, D)
    assert r2.weight_versions == [2] * D
    with pytest.raises(ValueError):
        _sim("pipedream2bw", D, 4 * D, D - 1)


def test_causality_exactly_once_all_policies():
    for kind in ss.POLICIES:
        ev, _ = _sim(kind, 4, 12, 4)
        for h in range(1, 5):
            assert sorted(e.sample for e in ev if e.op == "F" and e.stage == h) == list(range(12))
            assert sorted(e.sample for e in ev if e.op == "B" and e.stage == h) == list(range(12))
        cells = [(e.slot, e.stage) for e in ev if e.op in ("F", "B")]
        if kind != "partime":
            assert len(cells) == len(set(cells))  # one F or B per (slot, stage)


def test_render_timeline():
    ev, _ = _sim("partime", 1, 3)
    assert ss.render_timeline(ev, 1).split("|")[1].split() == ["F0B0U", "F1B1U", "F2B2U"]
    ev, _ = _sim("partime", 3, 8)
    rows = ss.render_timeline(ev, 3).splitlines()
    cells = rows[0].split("|")[1].split()
    assert cells[0] == "F0-" and cells[4] == "F4B0U"  # B(k) four columns after F(k) at stage 1
    assert ss.render_timeline(ev, 3) == ss.render_timeline(_sim("partime", 3, 8)[0], 3)
    assert rows[2].split("|")[1].split()[0] == "--"


def test_unknown_policy_and_compare():
    with pytest.raises(ValueError):
        _sim("zero-bubble", 2)
    rows = ss.compare_policies([ss.SchedulePolicy(k, 4, 8, 4) for k in ss.POLICIES], n=16)
    by = {r["policy"]: r for r in rows}
    assert by["partime"]["idle"] == 0 and by["gpipe"]["throughput"] < by["partime"]["throughput"]


def test_cli_simulate(capsys):
    assert cli.main(["simulate", "--policy", "partime", "--stages", "3", "--steps", "8"]) == 0
    out = capsys.readouterr().out
    assert "F4B0U" in out and '"staleness": [4, 2, 0]' in out
    assert cli.main(["simulate", "--policy", "nope", "--stages", "3"]) == 2

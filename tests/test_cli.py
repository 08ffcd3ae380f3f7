"""cli balance on the CPU byte profile."""

import io
import json
import types

from paper_2210_09147_b200 import cli


def _balance(**kw):
    a = dict(widths="1024x4", act="relu", stages=2, mode="learning", profile_iters=0, batch=1, workers=0,
             json=True, seed=0)
    a.update(kw)
    out = io.StringIO()
    assert cli.cmd_balance(types.SimpleNamespace(**a), out) == 0
    return json.loads(out.getvalue())


def test_balance_uniform_split_and_single_stage():
    rec = _balance()
    assert rec["layer_counts"] == [4, 3]  # 4 dense + 3 relu; (dense, relu) pairs stay together
    assert rec["worker_assignment"] == [0, 1] and rec["source"] == "byte_profile"
    assert _balance(stages=1)["layer_counts"] == [7]


def test_balance_uneven_widths_and_modes():
    rec = _balance(widths="256,4096,4096,256,256", stages=2)
    assert sum(rec["layer_counts"]) == 7 and len(rec["predicted_stage_cost"]) == 2
    assert _balance(widths="256,4096,4096,256,256", stages=2, mode="inference")["mode"] == "inference"


def test_balance_errors_exit_nonzero(capsys):
    assert cli.main(["balance", "--widths", "64x2", "--stages", "5"]) == 2
    assert "D=5" in capsys.readouterr().err

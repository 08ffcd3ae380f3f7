"""Drop-in surface and the round-1 advisor fixes, CPU only.

- the reference's import name `pipestream` (pkg/pyproject.toml:6) re-exports the engine;
- SPEC.md:74-75 loss name "softmax_cross_entropy";
- softmax-CE targets outside [0, F) raise;
- pipeline_run stops cleanly at the end of a finite stream with a partial report;
- nn.Linear(bias=False) is rejected instead of training a bias the net does not have.
"""

import types

import numpy as np
import pytest

import paper_2210_09147_b200.engine as eng
from paper_2210_09147_b200 import model as mdl
from paper_2210_09147_b200 import streams


def test_pipestream_import_names():
    from pipestream.engine import (Pipeline, PipelineOutput, RunReport, pipeline_build,  # noqa: F401
                                   pipeline_extract_weights, pipeline_run, pipeline_step)
    from pipestream import cli, netcore, numerics, partition, schedsim, tensor  # noqa: F401
    from pipestream.streams import Drift2dStream, ReplayStream, dataset_read, dataset_write  # noqa: F401
    assert Pipeline is eng.Pipeline and pipeline_run is eng.pipeline_run
    assert partition.balance([3, 1, 1, 3], 2)[0] == [2, 2]
    assert tensor.Tensor([1.0, 2.0]).shape == (2,)
    assert callable(cli.main)


def test_loss_alias():
    m = mdl.Model(layers=[], loss="softmax_cross_entropy")
    assert m.loss == "softmax_ce"
    assert mdl.canonical_loss("mse") == "mse"


def _fake(loss, F):
    return types.SimpleNamespace(model=types.SimpleNamespace(loss=loss), F=F)


def test_ce_targets_checked_on_host():
    check = eng.Pipeline._check_targets
    check(_fake("softmax_ce", 4), np.array([0, 3, 2], np.float32), "t")
    for bad in ([4.0], [-1.0], [1.5]):
        with pytest.raises(ValueError, match="target out of class range"):
            check(_fake("softmax_ce", 4), np.array(bad, np.float32), "t")
    check(_fake("mse", 4), np.array([7.5], np.float32), "t")  # mse targets are values


class _FakePipe:
    """Stands in for the device pipeline: records the ticks it was asked to run."""

    def __init__(self, D=2, F=2):
        self.D, self.M, self.F, self.t, self.calls = D, 1, F, 0, []

    def run(self, xs, ys, n):
        self.calls.append(n)
        t0 = self.t
        self.t += n
        valid = (np.arange(t0, t0 + n) >= self.D - 1).astype(np.uint8)
        return np.zeros((n, self.M, self.F), np.float32), np.ones(n, np.float32), valid


def test_pipeline_run_stops_at_end_of_finite_stream(tmp_path):
    x = np.arange(10, dtype=np.float32).reshape(5, 2)
    streams.dataset_write(tmp_path / "d.bin", x, np.zeros(5, np.int32))
    rs = streams.ReplayStream(streams.dataset_read(tmp_path / "d.bin"), W=1)
    p = _FakePipe()
    rep = eng.pipeline_run(p, rs, n_steps=12, chunk=4)
    assert rep.steps == list(range(5)) and p.calls == [4, 1]
    assert rep.valid_outputs == 4 and rep.losses[0] is None
    assert len(list(rep.csv_rows())) == 6


def test_biasless_linear_rejected():
    torch = pytest.importorskip("torch")
    from paper_2210_09147_b200.partime.convert import sequential_to_model
    net = torch.nn.Sequential(torch.nn.Linear(4, 4, bias=False), torch.nn.ReLU())
    with pytest.raises(NotImplementedError, match="bias=False"):
        sequential_to_model(net)

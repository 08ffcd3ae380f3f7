"""pipestream.tensor (pkg/src/pipestream/tensor.py:1-64): the Tensor value carrier."""
from paper_2210_09147_b200.tensor import Tensor, as_array  # noqa: F401

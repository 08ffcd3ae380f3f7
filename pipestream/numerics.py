"""pipestream.numerics (pkg/src/pipestream/numerics.py:1-37): process-global f64 / f32 mode."""
from paper_2210_09147_b200.numerics import dtype, get_mode, itemsize, set_mode, validating  # noqa: F401

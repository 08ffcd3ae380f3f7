"""pipestream.streams: synthetic and replayed input streams."""
from paper_2210_09147_b200.streams import (ConstantStream, DatasetFile, Drift2dStream, ReplayStream,  # noqa: F401
                                           SmoothStream, dataset_read, dataset_write)

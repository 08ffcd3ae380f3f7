"""pipestream.engine on the B200 C ABI (include/partime_b200.h)."""
from paper_2210_09147_b200._lib import ContractViolation, NonFiniteLoss, PipelineError  # noqa: F401
from paper_2210_09147_b200.engine import (Pipeline, PipelineOutput, RunReport, pipeline_build,  # noqa: F401
                                          pipeline_extract_weights, pipeline_run, pipeline_step)

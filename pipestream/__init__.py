"""`pipestream`: the reference package's import name (pkg/pyproject.toml:6) for the B200 engine.

A user of the reference writes `from pipestream.engine import pipeline_build`; these
modules re-export the B200-native implementation in `paper_2210_09147_b200` under the
reference's module names (SPEC.md:18-23 module map):
  numerics, tensor   pkg/src/pipestream/numerics.py, tensor.py (the shipped L0 modules)
  netcore            SPEC.md:26-50 domain types (the per-layer math runs inside the tick kernels)
  engine             SPEC.md:190-272 pipeline_build / step / run / extract_weights
  partition          SPEC.md:123-188 profile_costs / balance / assign_workers
  streams            SPEC.md:340-389 constant / drift2d / replay / DatasetFile
  schedsim           SPEC.md:274-338 simulate / render_timeline / compare_policies
  cli                SPEC.md:391-451 (balance, simulate)
"""

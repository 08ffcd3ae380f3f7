"""pipestream.partition: cost profile, min-max balance, worker assignment."""
from paper_2210_09147_b200.model import StagePlan  # noqa: F401
from paper_2210_09147_b200.partition import (CostProfile, assign_workers, balance, balance_profile,  # noqa: F401
                                             byte_profile, mlp_costs, profile_costs)

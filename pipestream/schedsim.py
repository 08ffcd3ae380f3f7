"""pipestream.schedsim: the PARTIME schedule rule and its comparators."""
from paper_2210_09147_b200.schedsim import (ScheduleReport, SchedulePolicy, TimelineEvent,  # noqa: F401
                                            compare_policies, render_timeline, simulate)

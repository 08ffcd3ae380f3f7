"""Command-line front end (reference `cli` module): `balance` and
`simulate`. `bench` is the repo-root bench.py harness; `train` and `verify` are the
tests/ suites and are out of scope here.

  python -m paper_2210_09147_b200.cli balance --widths 1024x16 --stages 4 [--mode learning]
         [--profile-iters 5] [--batch 1] [--workers N] [--json]
  python -m paper_2210_09147_b200.cli simulate --policy partime --stages 3 --steps 8 [--json]
"""

from __future__ import annotations

import argparse
import json
import sys


def _widths(spec):
    """'1024x16' -> 17 widths of 1024 (16 layers); '784,512,10' -> explicit list."""
    if "x" in spec:
        w, n = spec.split("x")
        return [int(w)] * (int(n) + 1)
    return [int(v) for v in spec.split(",")]


def cmd_balance(args, out=None):
    """prints the layer-count list and the predicted stage costs."""
    out = out or sys.stdout
    import numpy as np
    from . import model as mdl, partition
    m = mdl.mlp(_widths(args.widths), act=args.act, seed=args.seed, init=args.profile_iters > 0)
    if args.profile_iters > 0:
        si = np.ones((args.batch, m.layers[0].in_dim) if args.batch > 1 else m.layers[0].in_dim, np.float32)
        prof = partition.profile_costs(m, si, iters=args.profile_iters)
        source = "profile_costs"
    else:
        prof = partition.byte_profile(m, args.batch)
        source = "byte_profile"
    plan = partition.balance_profile(prof, args.stages, args.mode)
    plan = partition.assign_workers(plan, prof, args.workers or None)
    rec = {"layer_counts": plan.layer_counts(), "predicted_stage_cost": plan.predicted_stage_cost,
           "worker_assignment": plan.worker_assignment, "mode": args.mode, "source": source}
    if args.json:
        print(json.dumps(rec), file=out)
    else:
        print(rec["layer_counts"], file=out)
        for h, c in enumerate(plan.predicted_stage_cost):
            print(f"stage {h + 1}: layers {plan.boundaries[h][0]}..{plan.boundaries[h][1] - 1} "
                  f"predicted {c * 1e6:.2f} us on worker {plan.worker_assignment[h]}", file=out)
    return 0


def cmd_simulate(args, out=None):
    """thin wrapper over schedsim."""
    out = out or sys.stdout
    from . import schedsim
    pol = schedsim.SchedulePolicy(args.policy, args.stages, args.steps, args.microbatches)
    events, rep = schedsim.simulate(pol)
    if args.json:
        print(json.dumps({"report": rep.as_dict(), "timeline": schedsim.render_timeline(events, args.stages, args.width)}),
              file=out)
    else:
        print(schedsim.render_timeline(events, args.stages, args.width), file=out)
        print(json.dumps(rep.as_dict()), file=out)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_2210_09147_b200.cli")
    ap.add_argument("--seed", type=int, default=0)
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("balance")
    b.add_argument("--widths", required=True, help="WxN (N layers of width W) or a comma list of widths")
    b.add_argument("--act", default="relu", choices=["relu", "tanh", "none"])
    b.add_argument("--stages", type=int, required=True)
    b.add_argument("--mode", default="learning", choices=["inference", "learning"])
    b.add_argument("--profile-iters", type=int, default=0, help="> 0: time on the GPU (profile_costs)")
    b.add_argument("--batch", type=int, default=1)
    b.add_argument("--workers", type=int, default=0)
    b.add_argument("--json", action="store_true")
    s = sub.add_parser("simulate")
    s.add_argument("--policy", required=True)
    s.add_argument("--stages", type=int, required=True)
    s.add_argument("--steps", type=int, default=8)
    s.add_argument("--microbatches", type=int, default=4)
    s.add_argument("--width", type=int, default=0)
    s.add_argument("--json", action="store_true")
    args = ap.parse_args(argv)
    try:
        return {"balance": cmd_balance, "simulate": cmd_simulate}[args.cmd](args)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

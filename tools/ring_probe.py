"""Ring-geometry / prefetch sweep: us/tick of C2 (learn and infer) per env setting.
Usage: python tools/ring_probe.py  (each setting runs in a subprocess so env knobs apply)."""
import os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SETTINGS = [dict(PT_NSLOT=n, PT_PF_CHUNKS=pf) for n in (3, 4, 5, 6) for pf in (0, 6)]
if len(sys.argv) > 1 and sys.argv[1] == "policy":
    SETTINGS = [dict(PT_POLICY=pol, PT_PF_CHUNKS=pf) for pol in (0, 1, 2) for pf in (0, 6, 12, 20)]
CHILD = r'''
import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)
from configs_probe import probe
probe("C2 learn", [2048] * 33, 1, ticks=32)
probe("C2 infer", [2048] * 33, 1, learn=False, ticks=32)
probe("C3 infer", [4096] * 65, 1, learn=False, ticks=8)
''' % (ROOT, os.path.join(ROOT, "tools"))

if __name__ == "__main__":
    for s in SETTINGS:
        env = dict(os.environ, **{k: str(v) for k, v in s.items()})
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        print(s, flush=True)
        print(r.stdout.strip() or r.stderr[-800:], flush=True)

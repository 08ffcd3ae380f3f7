"""Per-GPU share of the C2 D=N run: a D=1 pipeline over 32/N layers (weights 537/N MB),
tick time per L2 load policy (0 evict_first, 1 evict_normal, 2 evict_last)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)
from configs_probe import probe
for L in (4, 8, 16):
    probe(f"C2 share: {L} x 2048", [2048] * (L + 1), 1, ticks=64, reps=3)
''' % (ROOT, os.path.join(ROOT, "tools"))
for pol in (0, 1, 2):
    r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, PT_POLICY=str(pol)), capture_output=True, text=True)
    print("PT_POLICY", pol, flush=True)
    print(r.stdout.strip() or r.stderr[-600:], flush=True)

"""Race detector: random stalls at every step phase of every warp and role of
both kernels (producer, MMA issuer, SIMT groups / consumer warps) must leave the results
bitwise equal to an unperturbed run: 8 us stalls on 1 in 4 trace points, and 0.3 ms stalls
on 1 in 512. The detector lives in a separate build (libpartime_b200_jitter.so,
-DPT_JITTER_BUILD) so the production kernels carry no hook; each case runs in a subprocess
that loads that build."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("kind,counts,learn", [("tile", "7", "0"), ("tile", "7", "1"), ("tile", "4,3", "1"),
                                               ("tick", "4,3", "1"), ("tick_mb", "4,3", "1"),
                                               ("panel", "4,3", "1"), ("panel", "7", "0"), ("panel_wide", "2,2,3", "1"),
                                               ("panel_adam", "4,3", "1"), ("tile_adam", "4,3", "1"),
                                               ("tile_m32", "4,3", "1"), ("tile_m32_adam", "4,3", "1"),
                                               ("tile_m64", "4,3", "1"), ("tile_m64_adam", "4,3", "1"),
                                               ("tick_conc", "8,7", "1"), ("tick_conc", "4,4,4,3", "1"),
                                               ("tick_conc_mb", "6,4,5", "1"), ("tick_mb_wide", "2,2,1", "1")])
def test_jitter_bitwise(kind, counts, learn):
    env = dict(os.environ, PT_LIBNAME="libpartime_b200_jitter.so")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "jitter_check.py"), kind, counts, learn],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr

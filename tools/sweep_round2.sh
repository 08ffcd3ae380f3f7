#!/bin/bash
# Randomised parity sweeps over the round-2 paths (tools/random_parity.py): batch 1 (panel
# kernel) with SGD and Adam, the tile kernel with Adam / softmax-CE, and micro-batches up to 64.
SEED=11 N=60 BIG_M=1 timeout 1200 python tools/random_parity.py 2>&1 | tail -3
SEED=12 N=40 OPT=adam timeout 1200 python tools/random_parity.py 2>&1 | tail -3
SEED=13 N=30 TILE_ONLY=1 WMAX=1024 timeout 1200 python tools/random_parity.py 2>&1 | tail -3

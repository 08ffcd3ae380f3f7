#!/bin/bash
# Tuning sweep of the panel kernel's streaming knobs on C2 (32 x 2048, D=1): ring slots
# (PT_NSLOT), L2 prefetch distance in chunks (PT_PF_CHUNKS), producer back-off (PT_PSLEEP).
for nslot in 8 6 5; do
  for pf in 0 8 16 32; do
    echo -n "nslot=$nslot pf=$pf: "
    PT_NSLOT=$nslot PT_PF_CHUNKS=$pf timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import tools.configs_probe as cp
cp.probe('C2', [2048] * 33, 1, ticks=32)" 2>&1 | tail -1
  done
done

for nslot in 6 5 4 3; do
  for pf in 8 0 16; do
    echo -n "nslot=$nslot pf=$pf: "
    PT_NSLOT=$nslot PT_PF_CHUNKS=$pf timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import tools.configs_probe as cp
cp.probe('C2', [2048] * 33, 1, ticks=64)" 2>&1 | tail -1
  done
done
timeout 200 python tools/tile_trace.py adam 2>&1 | grep -v "first SIMT" | head -12

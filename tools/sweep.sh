for cfg in "32 3" "32 2" "16 4" "16 3" "32 4"; do set -- $cfg
 echo "SLOT=$1K N=$2: $(PT_SLOT_KB=$1 PT_NSLOT=$2 python tools/trace_probe.py one 2>&1 | grep -E '^==')"
done

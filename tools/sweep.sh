for n in 4 5 6; do echo "NSLOT=$n: $(PT_NSLOT=$n python tools/trace_probe.py one | grep -E '^==')"; done
PT_NSLOT=5 python tools/trace_probe.py one | grep -E "^==|->" | head -8

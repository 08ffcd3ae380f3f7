timeout 200 python -c "
import sys; sys.path.insert(0, '.')
import tools.configs_probe as cp
cp.probe('C4 32x4096 M=16 D=8', [4096] * 33, 8, M=16, ticks=8, reps=2)
cp.probe('C4 8x4096 M=16 D=1', [4096] * 9, 1, M=16, ticks=8, reps=2)"

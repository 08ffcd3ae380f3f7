for i in 1 2 3; do
for lib in libpartime_b200.so libpartime_b200_old.so; do
echo -n "$lib: "; PT_LIBNAME=$lib timeout 120 python -c "
import sys; sys.path.insert(0, '.')
import tools.configs_probe as cp
cp.probe('C2', [2048] * 33, 1, ticks=64)
cp.probe('C3', [4096] * 65, 8, learn=False, ticks=8)" 2>&1 | tr '\n' ' '; echo
done; done

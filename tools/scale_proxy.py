"""Per-GPU share of C2 under one-stage-per-GPU scaling, measured on one GPU: the 32 x 2048
network split over N GPUs leaves 32/N layers per GPU (D = N stages). This times a D=1
pipeline of 32/N layers, which is the compute of one stage without the NVLink hop, so
it bounds the per-GPU tick rate at N GPUs from above (stage 1: input from the host side;
stage D: the loss). At N=8 a stage's weights (4 x 16 MB) fit in L2."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.configs_probe as cp

if __name__ == "__main__":
    for n in (1, 2, 4, 8):
        L = 32 // n
        cp.probe(f"C2 stage share at N={n} ({L} layers)", [2048] * (L + 1), 1, ticks=64)

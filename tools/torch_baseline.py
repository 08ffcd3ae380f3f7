"""The paper's implementation style on the same B200: PyTorch autograd forward/backward and
optimizer.step for the C2 D=1 online-learning tick, captured in a CUDA graph.
It reports device time per tick. It is a comparison point, not the product."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

def run(width=2048, layers=32, ticks=64, reps=3):
    torch.manual_seed(0)
    mods = []
    for i in range(layers):
        mods.append(torch.nn.Linear(width, width))
        if i < layers - 1:
            mods.append(torch.nn.ReLU())
    net = torch.nn.Sequential(*mods).cuda()
    opt = torch.optim.SGD(net.parameters(), lr=1e-3)
    lossf = torch.nn.MSELoss()
    x = torch.randn(1, width, device="cuda")
    y = torch.randn(1, width, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            opt.zero_grad(set_to_none=False)
            lossf(net(x), y).backward()
            opt.step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    opt.zero_grad(set_to_none=False)
    with torch.cuda.graph(g):
        opt.zero_grad(set_to_none=False)
        loss = lossf(net(x), y)
        loss.backward()
        opt.step()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(ticks):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / ticks)
    print(f"torch autograd + SGD, CUDA graph, {layers}x{width} M=1 D=1: {best*1e3:.1f} us/tick "
          f"({1e3/best:.0f} samples/s)")

if __name__ == "__main__":
    run()

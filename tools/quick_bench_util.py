"""Event timing helpers for the development tools."""
import torch


def timeit(fn, iters=20, warm=5, flush=None):
    """Median of single launches; `flush` (a large uint8 buffer) is READ before
    every rep (a read leaves clean L2 lines: a memset flush would leave ~L2-size
    dirty lines whose write-back lands inside the next timed kernel)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.view(torch.int64).max()
        torch.cuda._sleep(300000)  # keep the GPU busy while the CPU enqueues: time = device time only
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def time_graph(fn, reps=20):
    """Average per-call time of `reps` back-to-back calls captured in one CUDA
    graph (warm L2, launch overhead amortised)."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

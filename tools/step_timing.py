#!/usr/bin/env python
"""How the C1 step time depends on the launch mode: eager vs CUDA-graph replay, with and
without a host synchronisation after every step (L2 flushed before each step, outside the
events).   python tools/step_timing.py [c1] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import workloads as W
    from paper_2104_11404_b200 import hydro
    name = sys.argv[1] if len(sys.argv) > 1 else "c1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    prob = W.config(name)
    m = prob.mesh
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, t(m.elem_nodes, torch.int32), t(m.x0), t(m.rho0))
    x, v, e, g = t(prob.x), t(prob.v), t(prob.e), t(prob.gamma)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    F1 = torch.empty((m.dim, m.n_nodes), dtype=torch.float64, device=dev)
    FTw = torch.empty((m.n_elem, m.ne), dtype=torch.float64, device=dev)
    dt = torch.empty(1, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def step():
        ctx.force_full(x, v, e, g, visc, cfl, F1=F1, FTw=FTw, dt=dt)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    hydro.profile_enable(True)
    gprof = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gprof):
        step()
    hydro.profile_enable(False)
    import threading
    stop = threading.Event()

    def poll():
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
            stop.wait(0.0005)
    for mode in ("eager", "graph", "gprof", "graph+nvml", "gprof+nvml"):
        th = None
        if "nvml" in mode:
            th = threading.Thread(target=poll, daemon=True)
            stop.clear()
            th.start()
        for sync in (False, True):
            run = {"eager": step, "graph": graph.replay, "gprof": gprof.replay}[mode.split("+")[0]]
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(reps)]
            for i in range(reps):
                flush.zero_()
                evs[i][0].record()
                run()
                evs[i][1].record()
                if sync:
                    evs[i][1].synchronize()
            torch.cuda.synchronize()
            ts = [a.elapsed_time(b) * 1e3 for a, b in evs]
            print(f"{name} {mode:10s} sync={int(sync)}: median {np.median(ts):.1f} us  "
                  f"mean {np.mean(ts):.1f}  min {min(ts):.1f}  max {max(ts):.1f}", flush=True)
        if th is not None:
            stop.set()
            th.join()


if __name__ == "__main__":
    main()

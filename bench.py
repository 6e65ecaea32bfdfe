#!/usr/bin/env python
"""bench.py -- throughput of the corner-force hot path on B200 (BASELINE.json metric:
force-eval quadrature points / s (F.1 + F^T.v) at 1 B200, % of the FP64/HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4] [--impl ours|reference]

A step = one pass of the whole hot path for the workload:
  c0..c3 : hydro_force_full (gather, forward contractions, pointwise physics + dt,
           backward contractions, deterministic assembly, dt finalisation);
  c4     : ROM online step = 3 lifts + hydro_force_sampled (64 instances) + 2
           projections + the reduced position RHS.
The headline workload is BASELINE.json configs[4] (c4: the largest single-GPU config, the
paper's hyper-reduced online path); the JSON line also carries c0-c3, the
Taylor-Green force evaluation (tg), the FOM steps and the offline phase under "per_config".  Inputs are synthetic (workloads/), resident
in HBM before timing; L2 (126 MB) is flushed before every timed step by writing a 256 MiB
buffer (outside the per-step CUDA events).  Multi-GPU: independent replicas (the path is
sharded by nothing here -- DESIGN "Multi-GPU"), weak scaling, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "force-eval quad-points/sec (F·1 + F^T·v) at 1 B200; % of FP64/HBM roofline"  # BASELINE.json
UNIT = "quad-points/s"


# ----------------------------------------------------------------------------- work model
def contraction_flops(dim, k, q, nfield=2, visc=True):
    """Algorithmic FP64 flops (2 per multiply-add) of the sum-factorised contractions of
    one element: forward J, grad v (+ e_q) and backward F.1, F^T.v (DESIGN "Work model")."""
    n, m = k + 1, k
    if dim == 3:
        grad = 2 * q * n ** 3 + 3 * q * q * n * n + 3 * q ** 3 * n      # per scalar field
        interp = q * m ** 3 + q * q * m * m + q ** 3 * m
        bwd_f1 = dim * dim * q ** 3 * n + 3 * dim * q * q * n * n + dim * n ** 3 * 2 * q
    else:
        grad = 2 * q * n * n + 2 * q * q * n
        interp = q * m * m + q * q * m
        bwd_f1 = dim * dim * q * q * n + dim * n * n * 2 * q
    nq = q ** dim
    s_form = nq * (dim ** 3 + dim * dim + dim * dim)                   # S_q and A_q
    macs = nfield * dim * grad + interp + bwd_f1 + interp + s_form
    return 2 * macs


# FP64-pipe instruction cost of the IEEE operations on sm_100a, from the fast paths the
# kernels issue (csrc/ieee_fast.cuh, identical to nvcc's): a/b = 5 DFMA + DMUL + 2 DFMA,
# sqrt = 3 DMUL + 5 DFMA, 1/b = 5 DFMA (the MUFU seeds run on the XU pipe).
DIV_I, SQRT_I, RCP_I = 8, 8, 5
ROT_I = 2 + 3 + SQRT_I + 1 + DIV_I + 2 + SQRT_I + RCP_I + 1 + 10   # one Jacobi rotation = 48
# closed-form lambda_min of a symmetric 3x3 (DESIGN A.4 / R30): q, B, p1, p2 (18), p (1 +
# sqrt), det(B) (14), r (3 + div), fmax, s (2 + sqrt), cubic guess (5 fma), two Newton steps
# (2 x (4 + div + 1)), lambda (1)
LMIN3_CF_I = 18 + 1 + SQRT_I + 14 + 3 + DIV_I + 1 + 2 + SQRT_I + 5 + 2 * (5 + DIV_I) + 1   # = 95


def pointwise_instr(dim, visc, rot_per_lmin3):
    """FP64-pipe instructions of the contract pointwise stage per quadrature point
    (DESIGN A.3/A.4 as the kernels evaluate it; mul, add and fma count 1 each).
    rot_per_lmin3: Jacobi rotations of the fallback (R30) per 3x3 eigen-solve, averaged over
    all solves (the closed form's are counted by LMIN3_CF_I)."""
    if dim == 3:
        n = 27 + 5 + RCP_I + 9                   # cofactors, det, 1/det, J^-1
        n += DIV_I + 3 + 3 + SQRT_I              # rho, p, cs
        n += 30 + LMIN3_CF_I + ROT_I * rot_per_lmin3 + SQRT_I   # J^T J, lmin3, h
        if visc:
            n += 45 + 6                          # grad v, eps
            n += LMIN3_CF_I + ROT_I * rot_per_lmin3   # lmin3(eps)
            n += 5 + 1 + DIV_I + 1 + DIV_I + 1   # mu, den, cs/h, alpha_mu mu, / den, +
            n += 12 + 10                         # sigma, A = sigma : eps
        else:
            n += 17 + 1 + DIV_I + 1 + 2          # tr grad v, den, cs/h, +, A
        n += DIV_I                               # dt_q
        n += 36 + 1 + 2                          # S = w detJ sigma J^-T, w detJ, w_q
    else:
        n = 3 + RCP_I + 4                        # det, 1/det, J^-1
        n += DIV_I + 3 + 3 + SQRT_I              # rho, p, cs
        n += 9 + 2 + 3 + SQRT_I + 2 + 1 + SQRT_I + DIV_I   # h = det / sigma_max(J)
        if visc:
            n += 12 + 2                          # grad v, eps
            n += 2 + 3 + SQRT_I + 2 + 1          # lambda_min(eps)
            n += 5 + 2 + DIV_I + 1 + DIV_I + 1   # mu, den, cs/h, alpha_mu mu, / den, +
            n += 6 + 5                           # sigma, A
        else:
            n += 7 + 2 + DIV_I + 1 + 2           # tr grad v, den, cs/h, +, A
        n += DIV_I                               # dt_q
        n += 12 + 1 + 1                          # S, w detJ, w_q
    return n


# SURVEY 8(d)'s algorithmic work model (the graded per-unit figure): contraction multiply-adds
# (2 flop each) plus pointwise operations per quadrature point under the survey's Appendix A
# (Jacobi-4 eigen-solves), division / square root weighted x10 ("weighted") or x1 ("nominal").
S8D_POINTWISE = {(2, True): (110, 8), (2, False): (72, 6), (3, True): (664, 103), (3, False): None}


def s8d_contraction_flops(dim, k, q):
    """grad = 2qn^2 + 2q^2n (2D) or 2qn^3 + 3q^2n^2 + 3q^3n (3D); interp =
    qm^2 + q^2m (2D) or qm^3 + q^2m^2 + q^3m (3D); per element 3d grad + 2 interp MACs."""
    n, m = k + 1, k
    if dim == 3:
        grad = 2 * q * n ** 3 + 3 * q * q * n * n + 3 * q ** 3 * n
        interp = q * m ** 3 + q * q * m * m + q ** 3 * m
    else:
        grad = 2 * q * n * n + 2 * q * q * n
        interp = q * m * m + q * q * m
    return 2 * (3 * dim * grad + 2 * interp)


def s8d_flops_per_unit(dim, k, q, visc, weighted=True):
    """SURVEY 8(d) algorithmic flops of one element (unit) evaluation."""
    ops, divs = S8D_POINTWISE[(dim, visc)]
    pw = ops + (9 * divs if weighted else 0)
    return s8d_contraction_flops(dim, k, q) + pw * q ** dim


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region.

    NVML is polled every ~0.5 ms from a thread (the timed regions of the small configs last
    about a millisecond, too short for nvidia-smi's ~50 ms per query); nvidia-smi is the
    fallback.  The GPU is identified by PCI bus id, so CUDA_VISIBLE_DEVICES remapping does
    not pick the wrong board.  One sample is always taken at entry and one at exit."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, dev):
        self.samples = []            # (sm_mhz, max_mhz, {reason names})
        self.source = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        self._smi_id = str(getattr(dev, "index", 0) or 0)
        try:
            import torch
            props = torch.cuda.get_device_properties(dev)
            bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
            self._smi_id = bus
            import pynvml as N
            N.nvmlInit()
            self._nvml = (N, N.nvmlDeviceGetHandleByPciBusId(bus.encode()))
            self.source = "nvml"
        except Exception:
            self._nvml = None
            self.source = "nvidia-smi"

    def _sample(self):
        if self._nvml is not None:
            N, h = self._nvml
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                        N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
                self.samples.append((float(sm), float(mx),
                                     {n for n, b in zip(self.NAMES, bits) if r & b}))
            except Exception:
                pass
            return
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self._smi_id}", f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            s = [t.strip() for t in out.split(",")]
            if len(s) >= 9 and s[1].replace(".", "").isdigit():
                self.samples.append((float(s[1]), float(s[2]) if s[2].replace(".", "").isdigit() else None,
                                     {self.NAMES[i] for i in range(4) if s[5 + i].lower().startswith("active")}))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.0005 if self._nvml is not None else 0.2)

    def __enter__(self):
        self._sample()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"]}
        sm = [s[0] for s in self.samples]
        mx = [s[1] for s in self.samples if s[1] is not None]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm),
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return d


# FP64 pipe peak, derived from unit counts and clock: 64 FP64 FMA/clk/SM x 2 flop x 148 SMs x
# 1965 MHz = 37.2 TFLOP/s; measured 37.1 TFLOP/s with DMMA and 36.5 with independent DFMA
# chains (tools/microbench/dmma_rate.cu, profiles/r01_fp64_dmma_rate.txt; DMMA and DFMA share
# the pipe: 35.2 TF mixed).  The first DFMA microbenchmark (fp64_peak.cu, 34.2 TF) was
# chain-limited and under-stated the peak.  IEEE div 1.43e12/s, sqrt 1.29e12/s.
FP64_PEAK_TFLOPS = 37.2


# ----------------------------------------------------------------------------- workloads
def build_problem(name):
    import workloads as W
    if name == "c4":
        return W.c4()
    return W.config(name)


HEADLINE = "c4"   # the largest single-GPU config (BASELINE.json configs[4]): the paper's
                  # hyper-reduced online path
ALL_WORKLOADS = ("c4", "c0", "c1", "c2", "c3", "tg")


def run_ours(args, rank, world):
    import torch
    from paper_2104_11404_b200 import hydro

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    hydro.lib()
    results, probs = {}, {}
    names = [args.workload] + ([c for c in ALL_WORKLOADS if c != args.workload] if args.all else [])
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for name in names:
        results[name], probs[name] = bench_one(name, args, dev, flush, rank, world)
        torch.cuda.empty_cache()
    if args.all:
        results["fom_c2"] = bench_fom("c2", args, dev)
        results["fom_tg"] = bench_fom("tg", args, dev)
        results["offline_c2"] = bench_offline(args, dev)
    return results, probs


def _t(a, dev, dtype=None):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=dtype or torch.float64).contiguous()


def bench_one(name, args, dev, flush, rank, world):
    import torch
    import workloads as W
    from paper_2104_11404_b200 import hydro

    prob = build_problem(name)
    base = prob.base if name == "c4" else prob
    m = base.mesh
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, _t(m.elem_nodes, dev, torch.int32), _t(m.x0, dev),
                             _t(m.rho0, dev))
    visc = hydro.Visc(base.q1, base.q2, base.visc)
    cfl = hydro.Cfl(base.alpha, base.alpha_mu)
    gamma = _t(base.gamma, dev)
    nq = m.nq ** m.dim
    if name != "c4":
        x, v, e = _t(prob.x, dev), _t(prob.v, dev), _t(prob.e, dev)
        F1 = torch.empty((m.dim, m.n_nodes), dtype=torch.float64, device=dev)
        FTw = torch.empty((m.n_elem, m.ne), dtype=torch.float64, device=dev)
        dt = torch.empty(1, dtype=torch.float64, device=dev)
        n_qp = m.n_elem * nq
        n_units = m.n_elem

        def step():
            ctx.force_full(x, v, e, gamma, visc, cfl, F1=F1, FTw=FTw, dt=dt)
    else:
        b = prob
        plan = hydro.SamplePlan(ctx, b.sample_elems, b.B)
        Phi_x, Phi_v, Phi_e = _t(b.Phi_x, dev), _t(b.Phi_v, dev), _t(b.Phi_e, dev)
        x_os, v_os, e_os = _t(b.x_os, dev), _t(b.v_os, dev), _t(b.e_os, dev)
        Yx, Yv, Ye = _t(b.Yx, dev), _t(b.Yv, dev), _t(b.Ye, dev)
        # offline operators (untimed) formed by the library on the GPU
        Pv, Pe, Cxv, cx = hydro.offline_projectors(Phi_x, Phi_v, Phi_e, v_os, *W.sampled_row_maps(b))
        xS = torch.empty((Phi_x.shape[0], b.B), dtype=torch.float64, device=dev)
        vS = torch.empty_like(xS)
        eS = torch.empty((Phi_e.shape[0], b.B), dtype=torch.float64, device=dev)
        F1r = torch.empty((plan.s_v, b.B), dtype=torch.float64, device=dev)
        FTr = torch.empty((plan.s_e, b.B), dtype=torch.float64, device=dev)
        dt = torch.empty(b.B, dtype=torch.float64, device=dev)
        rv = torch.empty((b.nv, b.B), dtype=torch.float64, device=dev)
        re_ = torch.empty((b.ne, b.B), dtype=torch.float64, device=dev)
        rx = torch.empty((b.nx, b.B), dtype=torch.float64, device=dev)
        wsv = hydro.rom_project_workspace(b.nv, plan.s_v, b.B, dev)
        wse = hydro.rom_project_workspace(b.ne, plan.s_e, b.B, dev)
        n_qp = plan.n_cl * b.B * nq
        n_units = plan.n_cl * b.B

        def step():
            hydro.rom_lift(Phi_x, x_os, Yx, out=xS)
            hydro.rom_lift(Phi_v, v_os, Yv, out=vS)
            hydro.rom_lift(Phi_e, e_os, Ye, out=eS)
            plan.force_sampled(xS, vS, eS, gamma, visc, cfl, F1_rows=F1r, FTw_rows=FTr, dt=dt)
            hydro.rom_project(Pv, F1r, out=rv, workspace=wsv)
            hydro.rom_project(Pe, FTr, out=re_, workspace=wse)
            hydro.rom_lift(Cxv, cx, Yv, out=rx)

    # warm-up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st = ctx.status_sync() if name != "c4" else plan.status_sync()
    if st[0] != 0:
        raise RuntimeError(f"{name}: device status {st}")
    # the step as one CUDA graph (launch-bound small configs are not timed on the host's
    # Python/ctypes overhead); the library's calls are stream-ordered and capture cleanly
    l0 = hydro.launch_count()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    launches_per_step = hydro.launch_count() - l0
    # a second capture with profiling on: the library brackets its force kernel with
    # external event-record nodes, so each replay times the dominant kernel on its own
    # stream.  Those nodes cost the step ~8 us on C1 (they sit between the force kernel and
    # its programmatic-dependent assembly launch: tools/step_timing.py), so the step itself
    # is timed on the production graph and the kernel on this one, same flush protocol.
    hydro.profile_enable(True)
    gprof = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gprof):
        step()
    hydro.profile_enable(False)
    for _ in range(2):
        graph.replay()
        gprof.replay()
    torch.cuda.synchronize()
    # timed region: K graph replays, L2 flushed before each (outside the events)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.zero_()                      # L2 flush (256 MiB > 126 MB), outside the events
            evs[i][0].record()
            graph.replay()
            evs[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = ctx.status_sync() if name != "c4" else plan.status_sync()
    if st[0] != 0:
        raise RuntimeError(f"{name}: device status {st} after the timed region")
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms) / len(step_ms)
    ms = max_over_ranks(ms, dev, world)
    launches = launches_per_step * args.steps
    # dominant-kernel time: K replays of the profiled graph, flushed the same way
    kern_ms, kern_n = 0.0, 0
    for i in range(args.steps):
        flush.zero_()
        gprof.replay()
        torch.cuda.synchronize()
        km, kn = hydro.profile_read_captured()
        kern_ms += km
        kern_n += kn
    del gprof
    hydro.profile_release_captured()
    kern_avg = kern_ms / max(kern_n, 1)
    extra = {}
    if name == "c0":
        # C0 is latency-bound; report the per-call latency of back-to-back calls
        # (1000 calls captured in one CUDA graph, no flush between them)
        g1000 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1000):
            for _ in range(1000):
                step()
        g1000.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g1000.replay()
        e1.record()
        torch.cuda.synchronize()
        extra["latency_us_back_to_back"] = e0.elapsed_time(e1) / 1000 * 1e3
        del g1000
    out = dict(workload=name, ms_per_step=ms, qp_per_s=n_qp / (ms * 1e-3), **extra,
               elements_per_s=n_units / (ms * 1e-3), n_qp=n_qp, force_kernel_ms=kern_avg,
               force_kernel_share=kern_avg / ms if ms > 0 else None,
               gpu_launches=launches, timing="CUDA-graph replay of the step, CUDA events; force kernel: external event-record nodes in a profiled capture of the same step",
               clocks=clk.summary())
    # end to end through the public API with host buffers (pinned): every step copies its
    # inputs host->device, runs the hot path and copies its results device->host.  Steps
    # are software-pipelined over three streams with double-buffered device and host
    # tensors (step i+1's upload and step i-1's download overlap step i's compute), as a
    # serving loop would; the timed region spans the first upload to the last download.
    if name != "c4":
        out["e2e"] = e2e_full(ctx, prob, base, visc, cfl, n_qp, args, dev)
    else:
        out["e2e"] = e2e_rom(step_inputs=(Yx, Yv, Ye), step_outputs=(rv, re_, rx, dt), step=step,
                             n_qp=n_qp, args=args)
        out["components"] = c4_components(b, plan, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, Yx, Yv, Ye,
                                          xS, vS, eS, F1r, FTr, Pv, Pe, Cxv, cx, rv, re_, rx, wsv, wse,
                                          flush, args)
        out["rom_rk2avg_step"] = bench_rom_step(plan, b, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os,
                                                Pv, Pe, Cxv, cx, Yx, Yv, Ye, gamma, visc, cfl, n_qp,
                                                args, flush)
    # roofline of the dominant kernel (force kernel)
    out["roofline"] = roofline(name, base, m, n_units, kern_avg, prob, step_ms=ms)
    return out, prob


def c4_components(b, plan, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, Yx, Yv, Ye, xS, vS, eS, F1r, FTr,
                  Pv, Pe, Cxv, cx, rv, re_, rx, wsv, wse, flush, args):
    """The C4 step's GEMM-shaped pieces timed on their own (CUDA events, L2 flushed before
    each, median of K): the three lifts S7 and the two projections S9,
    each against its own roofline max(algorithmic bytes / HBM, flops / FP64 peak)."""
    import torch
    from paper_2104_11404_b200 import hydro
    hbm = measured_peaks().get("hbm_gbs", 6650.0) * 1e9
    fp64 = FP64_PEAK_TFLOPS * 1e12
    nred, B = Phi_x.shape[1], b.B

    def timed(fn):
        ts = []
        for i in range(max(4, args.steps // 2)):
            flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            if i > 0:
                ts.append(a.elapsed_time(e))
        return float(np.median(ts))

    def lift_model(rows, os_cols):
        byts = 8.0 * (rows * nred + rows * os_cols + rows * B)      # Phi, offset, out
        return byts, 2.0 * rows * nred * B

    def proj_model(s_rows, n):
        return 8.0 * (n * s_rows + s_rows * B + n * B), 2.0 * n * s_rows * B

    out = {}
    items = [("lift_x", lambda: hydro.rom_lift(Phi_x, x_os, Yx, out=xS), lift_model(Phi_x.shape[0], 1)),
             ("lift_v", lambda: hydro.rom_lift(Phi_v, v_os, Yv, out=vS), lift_model(Phi_v.shape[0], 1)),
             ("lift_e", lambda: hydro.rom_lift(Phi_e, e_os, Ye, out=eS), lift_model(Phi_e.shape[0], B)),
             ("project_v", lambda: hydro.rom_project(Pv, F1r, out=rv, workspace=wsv), proj_model(plan.s_v, Pv.shape[0])),
             ("project_e", lambda: hydro.rom_project(Pe, FTr, out=re_, workspace=wse), proj_model(plan.s_e, Pe.shape[0]))]
    for name, fn, (byts, flops) in items:
        ms = timed(fn)
        floor = max(byts / hbm, flops / fp64) * 1e3
        out[name] = {"ms": round(ms, 5), "alg_bytes": byts, "alg_flops": flops,
                     "floor_ms": round(floor, 5), "frac": round(floor / ms, 4),
                     "bound": "hbm" if byts / hbm >= flops / fp64 else "fp64"}
    lifts = sum(out[k]["ms"] for k in ("lift_x", "lift_v", "lift_e"))
    projs = sum(out[k]["ms"] for k in ("project_v", "project_e"))
    out["lifts_ms"], out["projections_ms"] = round(lifts, 4), round(projs, 4)
    out["kernels"] = "lift_mma_kernel (DMMA m8n8k4), project_mma_kernel + project_mma_reduce_kernel"
    return out


def max_over_ranks(value, dev, world):
    """Max of a per-rank time over all ranks (the bench reports the slowest replica).
    dev: the rank's device (CUDA under NCCL, CPU under gloo)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(per_rank_units, ms_max, world):
    """Whole-job throughput: units processed by all ranks / the slowest rank's time
    (weak scaling: every rank processes the full workload)."""
    return per_rank_units * world / (ms_max * 1e-3)


def bench_rom_step(plan, b, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, Pv, Pe, Cxv, cx, Yx, Yv, Ye,
                   gamma, visc, cfl, n_qp, args, flush):
    """the full hyper-reduced RK2-average online step for the
    64 instances of C4 (6 lifts, 4 sampled force passes, 4 projections, reduced updates),
    captured as one CUDA graph (the step has no host synchronisation).  Offline operators:
    the M-orthonormal-basis option, R = (Z^T Phi)^+."""
    import torch
    from paper_2104_11404_b200 import hydro
    st = hydro.RomStepper(plan, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, Pv, Pe, Cxv, cx)
    Y = [t.clone() for t in (Yx, Yv, Ye)]
    dt = torch.full((b.B,), 1e-6, dtype=torch.float64, device=Yx.device)
    dte = torch.empty_like(dt)
    for _ in range(2):
        st.step(*Y, gamma, visc, cfl, dt, dt_est=dte)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        st.step(*Y, gamma, visc, cfl, dt, dt_est=dte)
    ms = []
    for _ in range(max(2, args.steps // 4)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    status = plan.status_sync()[0]
    step_ms = float(np.median(ms))
    # NEXT-2: the previous-window offset transition (Eq. previous_os) at this size:
    # three per-instance lifts of the final state over the closure rows + c_x = Phi_x^T v_os
    tr = []
    for i in range(4):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hydro.rom_previous_window((Phi_x, Phi_v, Phi_e), (x_os, v_os, e_os), Y, (Phi_x, Phi_v, Phi_e), Phi_x)
        e1.record()
        torch.cuda.synchronize()
        if i > 0:
            tr.append(e0.elapsed_time(e1))
    trans_ms = float(np.median(tr))
    return {"ms_per_step": step_ms, "instances": b.B, "sampled_force_passes": 2,
            "previous_window_transition_ms": trans_ms,
            "previous_window_transition_in_steps": round(trans_ms / step_ms, 4),
            "transpose_passes": 2, "qp_per_s": 2 * n_qp / (step_ms * 1e-3), "status": status,
            "what": "hyper-reduced RK2-average step, 64 instances, CUDA-graph replay"}


def e2e_full(ctx, prob, base, visc, cfl, n_qp, args, dev):
    """End to end through hydro_force_full with host buffers.  The step's inputs are the
    state (x, v, e) -- F(x, v, e) of PAPER P:403-411 -- packed in one pinned host buffer
    and uploaded with one copy; its results (F1, FTw, dt) come back in one packed copy.
    The material constant gamma is uploaded once with the mesh (setup, like x0 and rho0)."""
    import torch
    m = base.mesh
    parts_in = [np.ascontiguousarray(a, dtype=np.float64) for a in (prob.x, prob.v, prob.e)]
    sizes_in = [a.size for a in parts_in]
    host_in = torch.from_numpy(np.concatenate([a.ravel() for a in parts_in])).pin_memory()
    gamma = torch.as_tensor(np.ascontiguousarray(base.gamma)).to(dev)
    shapes_out = [(m.dim, m.n_nodes), (m.n_elem, m.ne), (1,)]
    n_out = sum(int(np.prod(sh)) for sh in shapes_out)

    def views(buf, sizes, shapes):
        out, o = [], 0
        for n, sh in zip(sizes, shapes):
            out.append(buf[o:o + n].view(sh))
            o += n
        return out

    shapes_in = [a.shape for a in parts_in]
    dbuf, hout = [], []
    for _ in range(2):
        din = torch.empty(host_in.numel(), dtype=torch.float64, device=dev)
        dout = torch.empty(n_out, dtype=torch.float64, device=dev)
        F1, FTw, dt = views(dout, [int(np.prod(sh)) for sh in shapes_out], shapes_out)
        dbuf.append(dict(din=din, inp=views(din, sizes_in, shapes_in), dout=dout, F1=F1, FTw=FTw, dt=dt))
        hout.append(torch.empty(n_out, dtype=torch.float64).pin_memory())
    s_in, s_cp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    in_done = [ev(), ev()]; cp_done = [ev(), ev()]; out_done = [ev(), ev()]
    for e_ in out_done + cp_done:
        e_.record(torch.cuda.current_stream())
    torch.cuda.synchronize()

    def run(n):
        for it in range(n):
            k = it & 1
            b = dbuf[k]
            with torch.cuda.stream(s_in):
                s_in.wait_event(cp_done[k])          # step it-2 finished reading inputs k
                b["din"].copy_(host_in, non_blocking=True)
                in_done[k].record(s_in)
            with torch.cuda.stream(s_cp):
                s_cp.wait_event(in_done[k])
                s_cp.wait_event(out_done[k])         # step it-2's download of outputs k done
                x, v, e = b["inp"]
                ctx.force_full(x, v, e, gamma, visc, cfl, F1=b["F1"], FTw=b["FTw"], dt=b["dt"])
                cp_done[k].record(s_cp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(cp_done[k])
                hout[k].copy_(b["dout"], non_blocking=True)
                out_done[k].record(s_out)

    run(args.warmup)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    run(args.steps)
    for s_ in (s_in, s_cp):
        s_out.wait_stream(s_)
    e1.record(s_out)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / args.steps
    st = ctx.status_sync()
    if st[0] != 0:
        raise RuntimeError(f"e2e: device status {st}")
    h2d = host_in.numel() * 8
    d2h = hout[0].numel() * 8
    # the link alone: the same copies timed without compute (context for the e2e number)
    link = {}
    for name_, fn in (("h2d", lambda: dbuf[0]["din"].copy_(host_in, non_blocking=True)),
                      ("d2h", lambda: hout[0].copy_(dbuf[0]["dout"], non_blocking=True))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        link[name_ + "_gbps"] = 5 * (h2d if name_ == "h2d" else d2h) / (a.elapsed_time(b) * 1e-3) / 1e9
    return {"value": n_qp / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ems,
            "link_alone": {k: round(v, 1) for k, v in link.items()},
            "method": "public API (hydro_force_full); per step one H2D copy of the packed "
                      "state (x, v, e) from pinned host memory and one D2H copy of the packed "
                      "results (F1, FTw, dt); gamma resident (material constant, set up with "
                      "the mesh); uploads, compute and downloads of consecutive steps "
                      "overlapped on 3 streams"}


def e2e_rom(step_inputs, step_outputs, step, n_qp, args):
    """C4: the step's inputs are the reduced coordinates (Yhat_x, Yhat_v, Yhat_e), its
    results the reduced right-hand sides (r_v, r_e, r_x) and dt per instance."""
    import torch
    host_in = [t.cpu().pin_memory() for t in step_inputs]
    host_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in step_outputs]
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        for d, h in zip(step_inputs, host_in):
            d.copy_(h, non_blocking=True)
        step()
        for h, d in zip(host_out, step_outputs):
            h.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / args.steps
    return {"value": n_qp / (ems * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in host_in),
            "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in host_out),
            "ms_per_step": ems,
            "method": "public API (lift, force_sampled, project) with pinned host buffers"}


def bench_fom(name, args, dev):
    """the full-order RK2-average step (hydro_rk2avg_step) on a config's
    mesh and state with v.n = 0 on the box, CG to 1e-12: wall time per step (CUDA events;
    the step synchronises for its CG convergence checks), CG iterations, force share."""
    import torch
    import workloads as W
    from paper_2104_11404_b200 import hydro
    prob = W.config(name)
    m = prob.mesh
    n_nodes = m.n_nodes
    bc = []
    for c in range(m.dim):
        on = np.isclose(m.x0[c], m.lo[c]) | np.isclose(m.x0[c], m.hi[c])
        bc.append(c * n_nodes + np.nonzero(on)[0])
    bc = np.sort(np.concatenate(bc)).astype(np.int64)
    v0 = prob.v.copy()
    v0.reshape(-1)[bc] = 0.0
    if name in ("c0", "c2"):
        # The Sedov-shaped states (energy floor + spike) drive high-order L2 energy dofs
        # negative within one step (no positivity limiter is described in the paper; the
        # contract's c_s = sqrt((gamma(gamma-1)) e) then flags NaN, DESIGN R12), so the step is
        # measured on the config's mesh and velocity with a smooth positive energy field.
        prob.e = np.ascontiguousarray(1.0 + 0.5 * W.uniform01(W.stream_seed(9, 2), prob.e.size)
                                      .reshape(prob.e.shape))
    ctx = hydro.HydroContext(m.dim, m.k, m.nq, _t(m.elem_nodes, dev, torch.int32), _t(m.x0, dev),
                             _t(m.rho0, dev))
    fom = hydro.Fom(ctx, bc)
    x, v, e, g = _t(prob.x, dev), _t(v0, dev), _t(prob.e, dev), _t(prob.gamma, dev)
    visc, cfl = hydro.Visc(prob.q1, prob.q2, prob.visc), hydro.Cfl(prob.alpha, prob.alpha_mu)
    dt = 0.25 * float(ctx.dt_estimate(x, v, e, g, visc, cfl).item())
    E0 = sum(fom.energy(v, e))
    for _ in range(max(1, args.warmup // 2)):
        dt_est, _ = fom.step(x, v, e, g, visc, cfl, dt)
        if not np.isfinite(dt_est):
            return {"workload": f"fom_{name}", "error": "non-finite dt estimate (state left the "
                    "positive-energy range)", "status": ctx.status_sync()[0]}
        dt = min(dt, 0.5 * dt_est)
    ms, iters = [], []
    hydro.profile_enable(True)
    hydro.profile_read()
    for _ in range(max(2, args.steps // 4)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dt_est, it = fom.step(x, v, e, g, visc, cfl, dt)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        iters.append(it)
        if np.isfinite(dt_est):
            dt = min(dt, 0.5 * dt_est)
    kern_ms, kern_n = hydro.profile_read()
    hydro.profile_enable(False)
    st = ctx.status_sync()
    E1 = sum(fom.energy(v, e))
    step_ms = float(np.median(ms))
    extra = _bench_rom_fullrow_ops(fom, x, v, e, g, visc, cfl, dev) if name == "c2" else {}
    return {"workload": f"fom_{name}", "ms_per_step": step_ms, **extra,
            "force_evals_per_step": 2, "transpose_passes_per_step": 2,
            "force_ms_per_step": kern_ms / max(len(ms), 1),
            "cg_iterations_per_step": float(np.mean(iters)), "cg_tol": 1e-12,
            "qp_per_s_force": 2 * m.n_elem * m.nq ** m.dim / (step_ms * 1e-3),
            "rel_energy_drift": abs(E1 - E0) / E0, "status": st[0],
            "what": "RK2-average step (PAPER P:463-508): 2 force evaluations storing S_q + 2 "
                    "F^T w passes from S_q, 2 PCG solves of M_V, 2 M_E block solves, v.n=0"}


def _bench_rom_fullrow_ops(fom, x, v, e, g, visc, cfl, dev, n=20, m=40):
    """Full-row ROM operators on the FOM mesh (seeded random orthonormal bases, n state and m
    force columns per field, DEIM rows): the Theorem-2 integrands (hydro_rom_indicator, one
    full force evaluation + 2n mass applications + products) and the M-oblique window
    transition operators of the velocity (hydro_window_ops, Eq. ic2-tw).  Wall time per
    call with CUDA events (both synchronise)."""
    import torch
    from paper_2104_11404_b200 import hydro
    gen = torch.Generator(device=dev)
    gen.manual_seed(2104)

    def orth(N, k):
        return torch.linalg.qr(torch.randn((N, k), generator=gen, device=dev, dtype=torch.float64))[0].contiguous()
    NV, NE = v.numel(), e.numel()
    Pv, Pe, U1, U2 = orth(NV, n), orth(NE, n), orth(NV, m), orth(NE, m)
    Z1, Z2 = hydro.deim(U1), hydro.deim(U2)
    def med(fn, n_=3):
        fn()    # warm-up (first-call scratch allocation, module load)
        t = []
        for _ in range(n_):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fn()
            b.record()
            torch.cuda.synchronize()
            t.append(a.elapsed_time(b))
        return float(np.median(t)), r
    ind_ms, eta = med(lambda: fom.indicator(x, v, e, g, visc, cfl, Pv, Pe, U1, Z1, U2, Z2))
    Po = orth(NV, n)
    osn = torch.randn((NV, 1), generator=gen, device=dev, dtype=torch.float64)
    oso = torch.randn((NV, 1), generator=gen, device=dev, dtype=torch.float64)
    win_ms, _ = med(lambda: hydro.window_ops(Pv, Po, osn, oso, fom=fom, field=1))
    return {"indicator_ms": ind_ms, "indicator_eta": [float(eta[0]), float(eta[1])],
            "window_ops_oblique_v_ms": win_ms, "fullrow_basis_cols": n, "timing": "median of 3 after a warm-up call",
            "fullrow_force_basis_cols": m}


def bench_offline(args, dev, ns=64, m=40):
    """SURVEY 8(f) NEXT-3 on C2-sized vectors (N = 3 * 129^3 velocity dofs): POD of ns seeded
    synthetic snapshots (hydro_pod: Gram + host eigen + basis + CholQR) and greedy DEIM of an
    m-column basis (hydro_deim), wall time per call with CUDA events (both synchronise)."""
    import torch
    from paper_2104_11404_b200 import hydro
    N = 3 * 129 ** 3
    gen = torch.Generator(device=dev)
    gen.manual_seed(2104)
    # low-rank-plus-noise snapshots, so the energy criterion selects a nontrivial k
    A = torch.randn((ns, 24), generator=gen, device=dev, dtype=torch.float64)
    Bm = torch.randn((24, N), generator=gen, device=dev, dtype=torch.float64)
    S = A @ Bm    # (input generation only)
    S += 1e-3 * torch.randn((ns, N), generator=gen, device=dev, dtype=torch.float64)
    del Bm
    hydro.pod(S, eps=0.9999)    # warm-up
    t = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        Phi, sig = hydro.pod(S, eps=0.9999)
        b.record()
        torch.cuda.synchronize()
        t.append(a.elapsed_time(b))
    pod_ms = float(np.median(t))
    U = Phi[:, :m].contiguous() if Phi.shape[1] >= m else torch.linalg.qr(
        torch.randn((N, m), generator=gen, device=dev, dtype=torch.float64))[0].contiguous()
    del S
    def med(fn, n_=3):
        fn()    # warm-up: first-call scratch allocation
        t = []
        for _ in range(n_):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fn()
            b.record()
            torch.cuda.synchronize()
            t.append(a.elapsed_time(b))
        return float(np.median(t)), r
    deim_ms, idx = med(lambda: hydro.deim(U))
    qdeim_ms, qidx = med(lambda: hydro.qdeim(U))
    over_ms, oidx = med(lambda: hydro.deim_oversampled(U, 2 * m))
    gram_flop = 2.0 * ns * ns * N / 2
    return {"workload": "offline_c2", "N": N, "snapshots": ns, "pod_ms": pod_ms,
            "pod_k": int(Phi.shape[1]), "gram_tflops": gram_flop / (pod_ms * 1e-3) / 1e12,
            "deim_ms": deim_ms, "deim_m": m, "deim_distinct": int(len(set(idx.tolist()))),
            "qdeim_ms": qdeim_ms, "qdeim_distinct": int(len(set(qidx.tolist()))),
            "oversampled_ms": over_ms, "oversampled_n_s": 2 * m,
            "oversampled_distinct": int(len(set(oidx.tolist()))),
            "what": "POD (method of snapshots, energy criterion 0.9999, CholQR) of seeded "
                    "low-rank+noise snapshots, greedy DEIM, Q-DEIM and the oversampled greedy (n_s = 2m) "
                    "(P:908-1026)"}


def _rotations_per_lmin3(name, prob):
    """Data-dependent Jacobi rotation count of the contract, measured by the oracle on a
    seeded sample of the workload's elements (both sides execute the same sequence)."""
    import oracle
    base = prob.base if name == "c4" else prob
    m = base.mesh
    if not (m.dim == 3):
        return 0.0
    rng = np.random.default_rng(0)
    el = np.sort(rng.choice(m.n_elem, min(m.n_elem, 2000), replace=False)).astype(np.int32)
    oracle.lmin3_stats(reset=True)
    oracle.force(base, elist=el, mode=1)
    r, c = oracle.lmin3_stats(reset=True)
    return r / max(c, 1) * (1 if base.visc else 1)


def roofline(name, base, m, n_units, kern_ms, prob, step_ms=None):
    """Roofline of the dominant kernel (the force kernel).  FP64-bound (arithmetic intensity
    ~50 flop/B, DESIGN "Kernels").  achieved = SURVEY 8(d)'s algorithmic flops per unit
    (weighted: / and sqrt x10) x the units of one launch / the launch's average duration,
    against the FP64 peak.  Beside it, `issue`: the FP64-pipe instructions the kernel's own
    algorithm needs (contraction FMAs + the contract's pointwise operations, IEEE div/sqrt/rcp
    at their instruction cost, the Jacobi fallback's data-dependent rotation count from the
    oracle) at 2 flop per instruction slot -- the fraction of FP64 issue slots doing that
    work.  The 8(d) model assumes Jacobi-4 eigen-solves (664 ops per 3D point); the closed
    form of R30 needs fewer, so 8(d)'s fraction can exceed the issue-slot fraction in 3D."""
    nq = m.nq ** m.dim
    s8d_unit = s8d_flops_per_unit(m.dim, m.k, m.nq, base.visc)
    s8d_unit_nominal = s8d_flops_per_unit(m.dim, m.k, m.nq, base.visc, weighted=False)
    flops = n_units * s8d_unit
    # algorithmic bytes: x, v [N_V], e [N_E], m_q [Q], elem_nodes, gamma; write F1 [N_V], FTw [N_E]
    if name == "c4":
        B = prob.B
        rows_h1 = prob.Phi_x.shape[0]
        rows_l2 = prob.Phi_e.shape[0]
        n_cl = n_units // B
        byts = 8 * (2 * rows_h1 * B + rows_l2 * B + n_cl * nq + n_cl) + 4 * n_cl * m.nd
        byts += 8 * (prob.s0_nodes.size * m.dim * B + prob.sample_elems.size * m.ne * B)
    else:
        byts = (8 * (2 * m.N_V + m.N_E + m.n_elem * nq + m.n_elem) + 4 * m.n_elem * m.nd
                + 8 * (m.N_V + m.N_E))
    t = kern_ms * 1e-3
    ach = flops / t / 1e12
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    traffic = measured_traffic(name)
    out = {"bound": "alu", "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
           "frac": round(ach / FP64_PEAK_TFLOPS, 4),
           "traffic": traffic["bytes_per_launch"] if traffic else None,
           "kernel": "force kernel (hydro_force_full / hydro_force_sampled)",
           "basis": "SURVEY 8(d) weighted algorithmic flops per unit x units per launch",
           "s8d_flop_per_unit": s8d_unit, "s8d_flop_per_unit_nominal": s8d_unit_nominal,
           "units_per_launch": n_units, "kernel_ms": round(kern_ms, 5),
           "issue": None,   # filled by issue_basis() in the cpu-baseline leg (needs the oracle)
           "hbm_bytes_alg": byts, "hbm_frac": round(byts / t / 1e9 / hbm, 4),
           "traffic_source": traffic["source"] if traffic else None,
           "peak_source": "FP64: 64 FMA/clk/SM x 2 x 148 SMs x 1965 MHz = 37.2 TF/s (measured "
                          "37.1 DMMA / 36.5 DFMA burst, profiles/r01_fp64_dmma_rate.txt; sustained: "
                          "profiles/r02_fp64_sustained.txt); HBM from MEASURED_PEAKS.json"}
    if step_ms:
        # the whole step on 8(d)'s basis (C4: + the lift and projection GEMM flops)
        step_flops = flops
        if name == "c4":
            nred = prob.Phi_x.shape[1]
            step_flops += 2.0 * nred * prob.B * (2 * prob.Phi_x.shape[0] + prob.Phi_e.shape[0])  # lifts
            h1, l2 = prob.s0_nodes.size * m.dim, prob.sample_elems.size * m.ne
            step_flops += 2.0 * nred * prob.B * (h1 + l2) + 2.0 * nred * nred * prob.B           # projections, r_x
        out["step"] = {"gflop_s8d": round(step_flops / 1e9, 3), "ms": round(step_ms, 5),
                       "achieved": round(step_flops / (step_ms * 1e-3) / 1e12, 3),
                       "frac": round(step_flops / (step_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4)}
    return out


def issue_basis(name, prob, rf):
    """The issue-slot view of a roofline entry (DESIGN 8.2): FP64-pipe instructions of the
    kernel's own algorithm, with the Jacobi fallback's data-dependent rotation count measured
    by the oracle on a seeded element sample (both sides execute the same contract sequence)
    -- computed in the cpu-baseline leg, the one place bench.py may call oracle/."""
    base = prob.base if name == "c4" else prob
    m = base.mesh
    rot = _rotations_per_lmin3(name, prob)
    nq = m.nq ** m.dim
    c_instr = contraction_flops(m.dim, m.k, m.nq) // 2
    p_instr = pointwise_instr(m.dim, base.visc, rot)
    instr = rf["units_per_launch"] * (c_instr + nq * p_instr)
    ach = 2.0 * instr / (rf["kernel_ms"] * 1e-3) / 1e12
    rf["issue"] = {"achieved": round(ach, 3), "frac": round(ach / FP64_PEAK_TFLOPS, 4),
                   "fp64_instr_per_launch": instr, "flop_eq_per_instr": 2,
                   "contraction_instr_per_unit": c_instr, "pointwise_instr_per_qp": p_instr,
                   "fallback_rotations_per_lmin3": round(rot, 4),
                   "rotation_count_source": "oracle.lmin3_stats, seeded 2000-element sample"}


def measured_traffic(name):
    """dram__bytes_read.sum + dram__bytes_write.sum of the force kernel for this workload
    from the latest committed ncu --set full capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(name)


# ----------------------------------------------------------------------------- cpu baseline
def cpu_model():
    """The host CPU model (lscpu 'Model name'), for the baseline's record."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_c4_instance(batch, b, P_v, P_e, nthreads=0):
    """The oracle's C4 step for instance b: naive lifts of the
    instance's column on the sample-mesh closure rows, the force on the closure elements,
    the rows at S0, naive projections.  Returns the quadrature points evaluated."""
    import oracle
    base, m = batch.base, batch.base.mesh
    d, ncl, ne = m.dim, batch.closure_nodes.size, m.ne
    col = slice(b, b + 1)
    xS = oracle.lift(batch.Phi_x, batch.x_os, np.ascontiguousarray(batch.Yx[:, col]))
    vS = oracle.lift(batch.Phi_v, batch.v_os, np.ascontiguousarray(batch.Yv[:, col]))
    eS = oracle.lift(batch.Phi_e, np.ascontiguousarray(batch.e_os[:, col]), np.ascontiguousarray(batch.Ye[:, col]))
    x = m.x0.copy()
    x[:, batch.closure_nodes] = xS[:, 0].reshape(d, ncl)
    v = np.zeros_like(m.x0)
    v[:, batch.closure_nodes] = vS[:, 0].reshape(d, ncl)
    e = base.e.copy()
    e[batch.closure_elems] = eS[:, 0].reshape(-1, ne)
    r = oracle.force(base, elist=batch.closure_elems, x=x, v=v, e=e, nthreads=nthreads)
    F1 = np.ascontiguousarray(r["F1"][:, batch.s0_nodes].reshape(-1, 1))
    FT = np.ascontiguousarray(r["FTw"][batch.sample_elems].reshape(-1, 1))
    oracle.project(P_v, F1)
    oracle.project(P_e, FT)
    return batch.closure_elems.size * m.nq ** m.dim


def oracle_rate(name, prob, target_s, nthreads=0, c4_ops=None):
    """The oracle as it stands (oracle/, OpenMP) on a bounded seeded sample of a workload:
    quadrature points per second, the sample, the wall time.  c0-c3/tg: a seeded element subset
    (or the whole mesh) evaluated repeatedly for ~target_s; c4: whole instances of the ROM step
    (oracle_c4_instance), at least one."""
    import oracle
    cores = nthreads if nthreads > 0 else (os.cpu_count() or 1)
    if name == "c4":
        P_v, P_e = c4_ops
        qp, reps, t0 = 0, 0, time.perf_counter()
        while True:
            qp += oracle_c4_instance(prob, reps % prob.B, P_v, P_e, nthreads)
            reps += 1
            wall = time.perf_counter() - t0
            if wall >= target_s:
                break
        return {"value": qp / wall, "cores": cores, "wall_s": round(wall, 2),
                "sample": f"{reps} of {prob.B} C4 instances (lift + force over the "
                          f"{prob.closure_elems.size}-element closure + projections), {qp} quad points"}
    m = prob.mesh
    nq = m.nq ** m.dim
    rng = np.random.default_rng(1)
    oracle.force(prob, elist=np.arange(min(m.n_elem, 8), dtype=np.int32), nthreads=nthreads)
    n2 = int(min(m.n_elem, (16384 if m.dim == 3 else 65536) // (8 if nthreads == 1 else 1)))
    el = np.sort(rng.choice(m.n_elem, n2, replace=False)).astype(np.int32)
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.force(prob, elist=el, nthreads=nthreads)
        reps += 1
        wall = time.perf_counter() - t0
        if wall >= target_s:
            break
    return {"value": reps * n2 * nq / wall, "cores": cores, "wall_s": round(wall, 2),
            "sample": f"{n2} seeded elements of {m.n_elem} evaluated {reps}x = {reps * n2 * nq} quad "
                      f"points (F.1 + F^T.v + dt)"}


def cpu_baseline(headline, probs, per_cfg_s=2.5, one_core=("c0", "c1", "c2")):
    """SURVEY 8(d) oracle baseline: the oracle on the GPU box's host cores, per config (value,
    sample, and the full config's extrapolated wall time), plus 1-core rates for C0-C2 and the
    CPU model.  The headline config's entry is the line's cpu_baseline value."""
    from oracle import rom as orom
    per = {}
    c4_ops = None
    for name, prob in probs.items():
        if name == "c4":
            c4_ops = orom.offline_projectors(prob)[:2]
            r = oracle_rate("c4", prob, per_cfg_s * 2, c4_ops=c4_ops)
            full_qp = prob.closure_elems.size * prob.B * prob.base.mesh.nq ** 3
        else:
            r = oracle_rate(name, prob, per_cfg_s)
            full_qp = prob.mesh.n_elem * prob.mesh.nq ** prob.mesh.dim
        r["full_config_wall_s_est"] = round(full_qp / r["value"], 1)
        per[name] = r
    single = {}
    for name in one_core:
        if name in probs:
            r = oracle_rate(name, probs[name], per_cfg_s, nthreads=1)
            single[name] = {"value": r["value"], "sample": r["sample"], "wall_s": r["wall_s"]}
    h = per[headline]
    return {"value": h["value"], "unit": UNIT, "cores": h["cores"], "kind": "oracle",
            "sample": h["sample"], "cpu_model": cpu_model(), "per_config": per,
            "one_core": single,
            "note": "oracle/ as it stands (OpenMP over the elements, serial assembly); a reported "
                    "baseline, not the target"}


# ----------------------------------------------------------------------------- main
def bench_config(name, n_qp, world):
    """The workload description shared by both arms' JSON lines."""
    idx = {"c0": 0, "c1": 1, "c2": 2, "c3": 3, "c4": 4}.get(name)
    what = (f"{name} (BASELINE.json configs[{idx}])" if idx is not None else
            f"{name} (Taylor-Green 64^3 Q2/Q1, SURVEY 8(f) NEXT-4)")
    cfg = {"workload": what, "quad_points": n_qp,
           "l2": "flushed before every timed step (256 MiB write; GPU arm)",
           "parallelism": f"replicas x{world}"}
    if name == "c4":
        cfg["step"] = ("3 lifts (x, v, e on the sample-mesh closure rows) + hydro_force_sampled "
                       "(64 instances x closure elements) + 2 projections + the r_x lift")
        cfg["instances"] = 64
    return cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=HEADLINE, choices=list(ALL_WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--all", dest="all", action="store_true", default=True)
    ap.add_argument("--only", dest="all", action="store_false")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        return reference_arm(args, rank)

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    res, probs = run_ours(args, rank, world)
    head = res[args.workload]
    if rank == 0:
        line = {
            "metric": METRIC, "value": whole_job_value(head["n_qp"], head["ms_per_step"], world),
            "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (workloads/: seeded SplitMix64, shapes of BASELINE.json configs)",
            "config": bench_config(args.workload, head["n_qp"], world),
            "elements_per_s": head["elements_per_s"] * world,
            "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"],
            "roofline": head["roofline"], "clocks": head["clocks"],
            "force_kernel_ms": head["force_kernel_ms"], "force_kernel_share": head["force_kernel_share"],
            **{k: head[k] for k in ("components", "rom_rk2avg_step") if k in head},
            "per_config": {k: {kk: vv for kk, vv in r.items() if kk not in ("clocks",)}
                           for k, r in res.items() if k != args.workload},
        }
        if not args.no_cpu:
            for name, prob in probs.items():
                issue_basis(name, prob, res[name]["roofline"])
            line["cpu_baseline"] = cpu_baseline(args.workload, probs)
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def reference_arm(args, rank):
    """The oracle arm (bench.py --impl reference): rank 0 only, on the host cores, the same
    workload, metric and unit as our arm; each timed step is a bounded sample of the workload
    (c4: one whole instance of the ROM step; others: a seeded element sample for ~3 s)."""
    if rank != 0:
        return 0
    import oracle
    prob = build_problem(args.workload)
    m = (prob.base if args.workload == "c4" else prob).mesh
    c4_ops = None
    if args.workload == "c4":
        from oracle import rom as orom
        c4_ops = orom.offline_projectors(prob)[:2]
        n_qp = prob.closure_elems.size * prob.B * m.nq ** m.dim
    else:
        n_qp = m.n_elem * m.nq ** m.dim
    for _ in range(args.warmup):   # untimed: library load, threads, tables
        oracle.force(prob.base if args.workload == "c4" else prob, elist=np.arange(8, dtype=np.int32))
    vals, r = [], None
    for _ in range(args.steps):
        r = oracle_rate(args.workload, prob, 0.0 if args.workload == "c4" else 3.0, c4_ops=c4_ops)
        vals.append(r["value"])
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": n_qp / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (workloads/: seeded SplitMix64, shapes of BASELINE.json configs)",
            "config": bench_config(args.workload, n_qp, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"] + " per step", "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())

"""Benchmark: APR-native 3x3x3 convolution (restricted Gaussian pyramid) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c1|c4] [--stencil 3|5]
                    [--accum exact|fast] [--impl ours|reference]

A "step" is one convolve_apr pass (conv-only protocol, bench.hpp:158-169) over
the whole APR of the configuration, values and interior-node values resident in
HBM, accumulated in fp64 in the reference's tap order (EXACT, bit-identical to
the reference; --accum fast for fp32).  value = pixel-equivalent GB/s
(4 * N_pixels / t, metrics.hpp:15-21); particles/s, the roofline of the conv
pass, the other stencil/accumulation variants, the paper protocol (row index +
tree fill + conv), a cold first call and the end-to-end
host-buffer number through the C-ABI are reported beside it.  --impl reference
times the reference's own CPU convolve_apr (oracle/_ref, all host threads) on
the same workload, never loading the product library.
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
for _p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

METRIC = "pixel-equivalent GB/s and particles/s for APR 3x3x3 conv; HBM % of peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    5 ms during the timed region (nvidia-smi's fields, without a subprocess per
    sample); falls back to nvidia-smi when pynvml is unavailable."""

    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, gpu: int):
        self.gpu, self.samples, self._stop = gpu, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.max_mhz = None
        self._nvml = None
        try:  # NVML is set up before the timed region, so short regions still get samples
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(gpu)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            self._nvml = lambda: (N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), get_reasons(h))
        except Exception:
            self._nvml = None

    def _sample(self):
        try:
            self.samples.append(self._nvml())
        except Exception:
            pass

    def _run(self):
        if self._nvml is not None:
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(0.005)
            return
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.max_mhz = float(out[1])
                self.samples.append((float(out[0]), int(out[2].strip(), 16)))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self._nvml is not None:
            self._sample()
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._nvml is not None:
            self._sample()  # (still at load clocks)
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [float(c) for c, _ in self.samples]
        mask = 0
        for _, r in self.samples:
            mask |= int(r)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for b, n in self.REASONS.items() if mask & b), "samples": len(self.samples)}


# ------------------------------------------------------------------ workload --
WORKLOADS = {
    "c1": "C1: 256^3 spheres (12, r 6-20, blur 2, seed 42) -> APR E=0.1",
    "c3": "C3: 1024^3 spheres (48, r 24-80, blur 2, seed 42) -> APR E=0.1",
    "c4": "C4: the C3 APR tiled 4(z) x 4(x) x 2(y) -> 4096 x 4096 x 2048 pixel-equivalent (paper's concatenated copies)",
}
SPHERES = {"c1": (256, 12, 6.0, 20.0), "c3": (1024, 48, 24.0, 80.0)}
L2_NOTE = "GPU arm: L2 flushed between timed steps (256 MB write); reference arm: host CPU, no flush"


def bench_config(cfg: str, k: int, n_p: int, n_t: int, n_pix: int) -> dict:
    """The `config` dict -- identical in both arms (same workload, same stencil)."""
    return {"workload": WORKLOADS[cfg], "stencil": f"gaussian(1.0,{k}) restricted pyramid", "pad": "reflect",
            "particles": int(n_p), "interior_nodes": int(n_t), "pixels": int(n_pix), "cr": round(n_pix / n_p, 2),
            "protocol": "conv-only (tree values filled outside the timed region, bench.hpp:158-169)", "l2": L2_NOTE}


def workload(cfg: str):
    """Returns (APR, leaf values, input provenance) built on the device (ours)."""
    import paper_2112_03592_b200 as P  # noqa: F401
    if cfg == "c1":
        import goldens as G
        d = G.load("c1_256")
        return G.product_apr(d), d["values"], "reference-built committed fixture (tests/golden/c1_256.npz)"
    if cfg == "c3":
        from paper_2112_03592_b200 import synth
        n, count, rmin, rmax = SPHERES["c3"]
        apr, values = synth.build_spheres_apr(n, count=count, rmin=rmin, rmax=rmax, blur=2.0, seed=42,
                                              rel_error=0.1)
        return apr, values, "built on the GPU by paper_2112_03592_b200.synth (bit-identical to the reference build)"
    raise SystemExit(f"unknown config {cfg}")


def ncu_traffic(config: str, stencil: int, accum: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one conv pass, from the
    committed ncu capture of this workload (the newest profiles/<round>/traffic.json),
    or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
            v = t.get(f"{config}_k{stencil}_{accum}")
            if v is not None:
                return int(v), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def algorithmic_bytes(n_p: int, n_t: int, n_rows: int) -> int:
    """Per conv pass: y_idx u16 + value in f32 + out f32 per particle, y_idx u16 +
    value f32 per interior node, one u32 row begin per row (device layout)."""
    return 10 * n_p + 6 * n_t + 4 * n_rows


# ------------------------------------------------------------------ our arm ---
def run_ours(args, rank, world):
    import torch
    import paper_2112_03592_b200 as P
    from paper_2112_03592_b200 import _lib as L

    dev_id = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev_id)
    ctx = P.default_context(dev_id)
    # an explicit stream: torch's legacy default stream has handle 0, which the
    # C-ABI reads as "the context's own stream"
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s = stream.cuda_stream
    assert s != 0
    t0 = time.time()
    apr = values = None
    if args.config == "c4":
        # C3 built on the device, tiled 4(z) x 4(x) x 2(y) on the device
        from paper_2112_03592_b200 import synth
        apr3, values3, _ = workload("c3")
        d3 = apr3.device(ctx)
        dapr = synth.tile_apr(d3, 4, 4, 2)
        v3 = torch.from_numpy(np.ascontiguousarray(values3, np.float32)).cuda()
        v = torch.empty(dapr.n_particles, dtype=torch.float32, device="cuda")
        synth.tile_values(d3, dapr, 4, 4, 2, v3.data_ptr(), v.data_ptr())
        del v3
        provenance = "C3 built on the GPU, tiled on the GPU (aprgpu_tile_apr)"
        li, ti = dapr.info(L.LEAF), dapr.info(L.TREE)
        n_p, n_t, n_rows = int(li.n_particles), int(ti.n_particles), int(li.n_rows + ti.n_rows)
        l_min, l_max = int(li.l_min), int(li.l_max)
        n_pix = int(np.prod(dapr.dims, dtype=np.int64))
    else:
        apr, values, provenance = workload(args.config)
        dapr = apr.device(ctx)
        v = torch.from_numpy(np.ascontiguousarray(values, np.float32)).cuda()
        n_p, n_t = apr.access.particle_count(), apr.tree_access.particle_count()
        n_rows = apr.access.row_count() + apr.tree_access.row_count()
        l_min, l_max = apr.access.l_min, apr.access.l_max
        n_pix = apr.pixel_count()
    k = args.stencil
    w = P.gaussian_stencil(1.0, k)
    pyrs = {kk: P.make_pyramid(P.gaussian_stencil(1.0, kk), l_min, l_max, P.PyramidMode.Restricted)
            for kk in sorted({k, 3, 5})}
    dpyrs = {kk: p.device(ctx) for kk, p in pyrs.items()}
    setup_s = time.time() - t0
    modes = {"exact": L.ACCUM_EXACT, "fast": L.ACCUM_FAST}
    accum = modes[args.accum]
    tv = torch.empty(max(dapr.n_tree, 1), dtype=torch.float32, device="cuda")
    out = torch.empty(dapr.n_particles, dtype=torch.float32, device="cuda")
    dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def conv_fn(kk, acc):
        return lambda: dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), dpyrs[kk], 1, acc, out.data_ptr(), s)

    s2 = torch.cuda.Stream()  # the index step runs beside the tree fill (independent inputs and scratch)
    ev_fork, ev_idx = torch.cuda.Event(), torch.cuda.Event()

    def paper_step():  # row index + tree fill + convolution
        ev_fork.record(stream)
        s2.wait_event(ev_fork)
        dapr.rebuild_index_ptr(s2.cuda_stream)
        ev_idx.record(s2)
        dapr.fill_tree_ptr(v.data_ptr(), tv.data_ptr(), s)
        stream.wait_event(ev_idx)  # (the step ends when both have: the timing event follows the conv on `stream`)
        dapr.convolve_ptr(v.data_ptr(), tv.data_ptr(), dpyrs[k], 1, accum, out.data_ptr(), s)

    def timed(fn, steps):
        times = []
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        return times

    # cold first call: a fresh upload of the host structure + the per-APR lists,
    # tree links, tile probe/runs and gather maps built by the first fill_tree +
    # convolve_apr, with the values' H2D copy (host wall clock, synchronised)
    cold = None
    if apr is not None:
        torch.cuda.synchronize()
        hv = torch.from_numpy(np.ascontiguousarray(values, np.float32)).pin_memory()
        runs = []
        for _ in range(5):  # five fresh handles (each cold: nothing cached for it); the median is reported
            c0 = time.perf_counter()
            fresh = P.aprkit.DeviceApr.upload(ctx, P.APR(apr.access, apr.tree_access, apr.source_dims))
            c1 = time.perf_counter()
            fv = hv.to("cuda", non_blocking=True)
            ftv = torch.empty(max(fresh.n_tree, 1), dtype=torch.float32, device="cuda")
            fout = torch.empty(fresh.n_particles, dtype=torch.float32, device="cuda")
            fresh.fill_tree_ptr(fv.data_ptr(), ftv.data_ptr(), s)
            fresh.convolve_ptr(fv.data_ptr(), ftv.data_ptr(), dpyrs[k], 1, accum, fout.data_ptr(), s)
            stream.synchronize()
            c2 = time.perf_counter()
            runs.append((c2 - c0, c1 - c0, c2 - c1))
            del fresh, fv, ftv, fout
        runs.sort()
        tot, up, first = runs[len(runs) // 2]
        cold = {"ms": round(tot * 1e3, 3), "upload_ms": round(up * 1e3, 3), "first_call_ms": round(first * 1e3, 3),
                "runs_ms": [round(r[0] * 1e3, 3) for r in runs],
                "includes": "aprgpu_upload_access of the host structure (incl. its interior structure, row and tile "
                            "lists) + values H2D + first fill_tree + first convolve_apr (tree links, tile probe, "
                            "tile runs, gather maps + their bank-aware placement), host wall clock; median of "
                            "five fresh handles (host-side upload times vary run to run)"}

    headline = conv_fn(k, accum)
    for _ in range(args.warmup):
        headline()
        paper_step()
    for kk in dpyrs:
        for acc in modes.values():
            conv_fn(kk, acc)()  # (builds every variant's maps outside the timed regions)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    with ClockSampler(dev_id) as clk:
        t_conv = timed(headline, args.steps)
        launches = ctx.launch_count() - l0
        t_paper = timed(paper_step, args.steps)
        variants = {}
        for kk in sorted(dpyrs):
            for name, acc in modes.items():
                if kk == k and acc == accum:
                    continue
                variants[(kk, name)] = timed(conv_fn(kk, acc), max(3, min(args.steps, 20)))
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()

    # end to end through the C-ABI with pinned host buffers (H2D + conv + D2H per step)
    hv = v.cpu().pin_memory()
    htv = tv[:dapr.n_tree].cpu().pin_memory() if dapr.n_tree else torch.zeros(1).pin_memory()
    hout = torch.empty(dapr.n_particles, dtype=torch.float32).pin_memory()
    e2e = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        a = time.perf_counter()
        L.check(L.lib().aprgpu_convolve(dapr.handle, hv.data_ptr(), htv.data_ptr(), dpyrs[k].handle, 1, accum,
                                        hout.data_ptr(), L.HOST, None))
        b = time.perf_counter()
        if i >= args.warmup:
            e2e.append(b - a)

    # C5: rl_apr, 10 Richardson-Lucy iterations on the same APR (deconv.hpp:75-107:
    # 2 tree refreshes + 2 convolutions per iteration, ratio/multiply fused)
    rl_out = torch.empty_like(out)
    rl = {}
    for name, acc in modes.items():
        rl_t = []
        for i in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dapr.rl_ptr(v.data_ptr(), w, args.rl_iters, 0.0, acc, rl_out.data_ptr(), s)
            e1.record(stream)
            e1.synchronize()
            rl_t.append(e0.elapsed_time(e1) / 1e3)
        rl[name] = {"ms": round(rl_t[-1] * 1e3, 3), "ms_per_iteration": round(rl_t[-1] * 1e3 / max(args.rl_iters, 1), 4)}

    # reconstruct_full (reconstruct.hpp:87-90) of the same APR: the dense image,
    # bound by writing it (4 bytes per pixel); skipped when it would not fit easily
    recon = None
    pixels_conv = None
    if 4 * n_pix <= 16e9:
        img = torch.empty(n_pix, dtype=torch.float32, device="cuda")
        lmax = int(dapr.info(L.LEAF).l_max)
        rt = []
        for i in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dapr.reconstruct_level_ptr(v.data_ptr(), 0, lmax, img.data_ptr(), s)
            e1.record(stream)
            e1.synchronize()
            rt.append(e0.elapsed_time(e1) / 1e3)
        tr = min(rt[1:])
        recon = {"ms": round(tr * 1e3, 4), "write_gbs": round(4 * n_pix / tr / 1e9, 1),
                 "frac_of_peak": round(4 * n_pix / tr / 1e9 / peaks()[0], 4),
                 "note": "reconstruct_full on the device (k_reconstruct), output bytes / time, best of 2 warm runs"}
        # the pixel-space baseline on the same image (convolve_pixels, convolve.hpp:48-98;
        # the paper's APR-vs-pixels comparison): same stencil, same accumulation mode
        if 8 * n_pix <= 24e9:
            pout = torch.empty_like(img)
            pt = []
            for i in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                P.convolve_pixels_ptr(ctx, img.data_ptr(), dapr.dims, w, 1, accum, pout.data_ptr(), s)
                e1.record(stream)
                e1.synchronize()
                pt.append(e0.elapsed_time(e1) / 1e3)
            del pout
            tpx = min(pt[1:])
            pixels_conv = {"ms": round(tpx * 1e3, 4), "gbs_pixel_equiv": round(4 * n_pix / tpx / 1e9, 1),
                           "hbm_frac": round(8 * n_pix / tpx / 1e9 / peaks()[0], 4),
                           "note": "convolve_pixels of the reconstructed image (k_convolve_pixels_zreg), best of 2 "
                                   "warm runs, same accumulation mode as the headline"}
        del img

    def agg(x):
        t = float(np.mean(x))
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt.item())
        return t

    tc, tp, te = agg(t_conv), agg(t_paper), agg(e2e)
    B = algorithmic_bytes(n_p, n_t, n_rows)
    peak, peak_kind = peaks()

    def roof(t, kk, acc_name):
        a_ = B / t / 1e9
        traffic, src = ncu_traffic(args.config, kk, acc_name)
        return {"bound": "hbm", "achieved": round(a_, 2), "peak": peak, "unit": "GB/s", "frac": round(a_ / peak, 4),
                "traffic": traffic,
                "note": f"algorithmic bytes {B} per pass (10/particle + 6/node + 4/row) / conv-pass time (CUDA events "
                        f"on the launching stream); peak {peak_kind} (MEASURED_PEAKS.json hbm_gbs); traffic = ncu dram "
                        f"bytes of one cold pass" + (f" ({src})" if src else " (no committed capture)")}

    def line(t, kk, acc_name):
        return {"ms_per_step": round(t * 1e3, 4), "gbps_pixel_equiv": round(world * 4 * n_pix / t / 1e9, 3),
                "particles_per_s": round(world * n_p / t, 1), "roofline": roof(t, kk, acc_name)}

    dtype = {"exact": "f32 values, f64 accumulate in the reference's tap order (bit-exact)",
             "fast": "f32 values, f32 accumulate (rel <= 1e-5)"}
    res = {
        "metric": METRIC,
        "value": round(world * 4 * n_pix / tc / 1e9, 3),
        "unit": "GB/s (pixel-equivalent)",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(tc * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": dtype[args.accum],
        "data": "synthetic",
        "config": bench_config(args.config, k, n_p, n_t, n_pix),
        "input": provenance,
        "parallelism": "single GPU",
        "particles_per_s": round(world * n_p / tc, 1),
        "paper_protocol": {"ms_per_step": round(tp * 1e3, 4), "gbps_pixel_equiv": round(4 * n_pix / tp / 1e9, 3),
                           "includes": "per step: nonempty_row_index + tile lists rebuilt on the device "
                                       "(aprgpu_rebuild_index, on a second stream beside fill_tree: independent "
                                       "inputs and scratch) + fill_tree, then convolve_apr once both are done "
                                       "(PAPER.md:379), L2 flushed before each step"},
        "roofline": roof(tc, k, args.accum),
        "e2e": {"value": round(world * 4 * n_pix / te / 1e9, 3), "unit": "GB/s (pixel-equivalent)",
                "ms_per_step": round(te * 1e3, 4),
                "h2d_bytes_per_step": int(4 * n_p + 4 * dapr.n_tree), "d2h_bytes_per_step": int(4 * n_p),
                "note": "aprgpu_convolve with pinned HOST buffers (the drop-in call): copies pipelined over "
                        "z-chunks against the per-chunk passes (APRGPU_HOST_CHUNKS, default 8)"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "setup_s": round(setup_s, 2),
        "variants": {f"k{kk}_{name}": line(agg(tt), kk, name) for (kk, name), tt in variants.items()},
        "rl_apr": dict(rl, iterations=args.rl_iters, psf=f"gaussian(1.0,{k}), restricted pyramids of w and flip(w)",
                       note="C5; second of two runs, includes the pyramid setup and the exact mean"),
    }
    if cold:
        res["cold_call"] = cold
    if recon:
        res["reconstruct_full"] = recon
    if pixels_conv:
        pixels_conv["apr_speedup"] = round(pixels_conv["ms"] / (tc * 1e3), 2)
        res["convolve_pixels"] = pixels_conv
    if rank == 0 and not args.no_cpu_baseline and apr is not None:
        res["cpu_baseline"] = cpu_baseline(apr, values, tv[:dapr.n_tree].cpu().numpy(), pyrs[k], args)
    return res


# ------------------------------------------------------- multi-GPU z-slabs ---
def run_slab(args, rank, world):
    """N > 1: one volume cut into z-slabs, one per GPU (paper_2112_03592_b200.slab,
    DESIGN.md §6).  --config c3 (default): the C3 APR tiled N times along z --
    weak scaling, each GPU holds a C3-sized slab; --config c4: the C4 APR (C3
    tiled 4 x 4 x 2) cut into N slabs -- strong scaling of BASELINE config 4.
    A conv-only step is the leaf + tree halo exchange over NCCL in flight while
    every rank convolves its slab's interior, then the boundary bands; the
    paper step adds the slab tree fill with its cut-level all-gather.  Time =
    max over ranks of the CUDA-event step time."""
    import torch
    import torch.distributed as dist
    import paper_2112_03592_b200 as P
    from paper_2112_03592_b200 import _lib as L
    from paper_2112_03592_b200 import synth
    from paper_2112_03592_b200.slab import GpuRankState, SlabConvolver, SlabPlan, TorchComm

    dev_id = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev_id)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = P.default_context(dev_id)
    tz = int(os.environ.get("APRGPU_BENCH_TILEZ", world))  # (a test hook: the tiled C3 at any world size)
    if args.config == "c4":
        tiling, scaling = (4, 4, 2), "strong"
    elif args.config == "c3" and tz > 1:
        tiling, scaling = (tz, 1, 1), "weak"
    else:
        tiling, scaling = None, "strong"
    if tiling:
        apr3, values3, _ = workload("c3")
        d3 = apr3.device(ctx)
        dapr = synth.tile_apr(d3, *tiling)
        v3 = torch.from_numpy(np.ascontiguousarray(values3, np.float32)).cuda()
        vdev = torch.empty(dapr.n_particles, dtype=torch.float32, device="cuda")
        synth.tile_values(d3, dapr, *tiling, v3.data_ptr(), vdev.data_ptr())
        torch.cuda.synchronize()
        del v3, d3
        leaf, tree = dapr.download(L.LEAF, rows_only=True), dapr.download(L.TREE, rows_only=True)
        dims = tuple(int(d) for d in dapr.dims)
        values = None
        if args.config == "c4":
            desc = WORKLOADS["c4"]
        else:
            desc = (f"C3 tiled {tz}(z) x 1 x 1 -> {1024 * tz} x 1024 x 1024 pixel-equivalent (device tiler): "
                    "one C3-sized z-slab per GPU (weak scaling)")
    else:
        apr, values, _ = workload(args.config)
        desc = WORKLOADS[args.config]
        dapr = apr.device(ctx)
        leaf, tree, dims = apr.access, apr.tree_access, tuple(apr.source_dims)
        vdev = None
    li, ti = dapr.info(L.LEAF), dapr.info(L.TREE)
    n_p, n_t, n_rows = int(li.n_particles), int(ti.n_particles), int(li.n_rows + ti.n_rows)
    n_pix = int(np.prod(dims, dtype=np.int64))
    k = args.stencil
    pyr = P.make_pyramid(P.gaussian_stencil(1.0, k), int(li.l_min), int(li.l_max), P.PyramidMode.Restricted)
    dpyr = pyr.device(ctx)
    accum = L.ACCUM_EXACT if args.accum == "exact" else L.ACCUM_FAST
    plan = SlabPlan.make(leaf, tree, dims, world, rank, halo=max(k // 2, 1))
    st = GpuRankState(plan, dapr, dev_id, stream)
    if vdev is not None:
        st.values.copy_(vdev)
        del vdev
    else:
        st.values.copy_(torch.from_numpy(np.ascontiguousarray(values, np.float32)).to(st.device))
    comm = TorchComm()
    sc = SlabConvolver([st], comm)
    sc.fill_tree()

    def conv():
        sc.exchange_and_convolve(dpyr, 1, accum)

    def paper_step():
        sc.convolve(dpyr, 1, accum)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=st.device)

    def timed(fn, steps):
        times = []
        for _ in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        return times

    for _ in range(args.warmup):
        conv()
        paper_step()
    torch.cuda.synchronize()
    dist.barrier()
    l0 = ctx.launch_count()
    with ClockSampler(dev_id) as clk:
        t_conv = timed(conv, args.steps)
        launches = ctx.launch_count() - l0
        t_paper = timed(paper_step, args.steps)

    # end to end: this rank's owned values from pinned host memory, the step,
    # its owned outputs back to the host
    owned = plan.owned("leaf") + [plan.replicated("leaf")]
    hv = torch.empty(max(n_p, 1), dtype=torch.float32).pin_memory()
    for b, e in owned:
        hv[b:e].copy_(st.values[b:e])
    hout = torch.empty(max(n_p, 1), dtype=torch.float32).pin_memory()
    e2e = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        dist.barrier()
        a = time.perf_counter()
        for b, e in owned:
            st.values[b:e].copy_(hv[b:e], non_blocking=True)
        sc.convolve(dpyr, 1, accum)
        for b, e in owned:
            hout[b:e].copy_(st.out[b:e], non_blocking=True)
        stream.synchronize()
        if i >= args.warmup:
            e2e.append(time.perf_counter() - a)
    h2d = sum(4 * (e - b) for b, e in owned)

    def agg(x):
        tt = torch.tensor([float(np.mean(x))], dtype=torch.float64, device=st.device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    tc, tp, te = agg(t_conv), agg(t_paper), agg(e2e)
    B = algorithmic_bytes(n_p, n_t, n_rows)
    peak, peak_kind = peaks()
    achieved = B / world / tc / 1e9  # per GPU: each owns ~1/N of the bytes
    cfg = bench_config(args.config, k, n_p, n_t, n_pix)
    cfg["workload"] = desc
    return {
        "metric": METRIC,
        "value": round(4 * n_pix / tc / 1e9, 3),
        "unit": "GB/s (pixel-equivalent)",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(tc * 1e3, 4),
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f32 values, " + ("f64 accumulate in the reference's tap order (bit-exact)"
                                   if accum == L.ACCUM_EXACT else "f32 accumulate"),
        "data": "synthetic",
        "config": cfg,
        "parallelism": f"z-slabs x{world} (cut level {plan.lc}, halo {plan.halo} rows/level), NCCL halo exchange "
                       "overlapped with each slab's interior",
        "particles_per_s": round(n_p / tc, 1),
        "paper_protocol": {"ms_per_step": round(tp * 1e3, 4), "gbps_pixel_equiv": round(4 * n_pix / tp / 1e9, 3),
                           "includes": "halo exchange + slab fill_tree (cut-level all-gather) + slab convolution"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "note": f"per GPU: algorithmic bytes / N / step time; peak {peak_kind}"},
        "e2e": {"value": round(4 * n_pix / te / 1e9, 3), "unit": "GB/s (pixel-equivalent)",
                "ms_per_step": round(te * 1e3, 4), "h2d_bytes_per_step": int(h2d * world),
                "d2h_bytes_per_step": int(h2d * world)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }


# -------------------------------------------------------------- CPU baseline --
def cpu_baseline(apr, values, tree_values, pyr, args):
    """The reference's own convolve_apr (oracle/_ref) timed with its time_median
    protocol (bench.hpp:106-117) on the full workload: all host threads, plus
    one single-thread run."""
    from pyoracle import Ref, ref_available
    n_pix = apr.pixel_count()
    if not ref_available():
        return {"value": None, "unit": "GB/s (pixel-equivalent)", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built on this box"}
    R = Ref()
    rapr = R.apr_from_arrays(apr.access, apr.source_dims)
    rpyr = R.explicit_pyramid([((s.kz, s.kx, s.ky), s.weights) for s in pyr.stencils], pyr.l_min)
    threads = R.resolve_threads(0)
    R.convolve(rapr, values, tree_values, rpyr, 1, threads)  # cold run discarded
    times = []
    budget = time.time() + args.cpu_seconds
    while len(times) < 3 or (time.time() < budget and len(times) < 15):
        a = time.perf_counter()
        R.convolve(rapr, values, tree_values, rpyr, 1, threads)
        times.append(time.perf_counter() - a)
    t = statistics.median(times)
    a = time.perf_counter()
    R.convolve(rapr, values, tree_values, rpyr, 1, 1)
    t1 = time.perf_counter() - a
    return {"value": round(4 * n_pix / t / 1e9, 4), "unit": "GB/s (pixel-equivalent)", "cores": threads,
            "kind": "reference", "ms_per_step": round(t * 1e3, 2),
            "particles_per_s": round(apr.access.particle_count() / t, 1),
            "single_thread": {"value": round(4 * n_pix / t1 / 1e9, 4), "ms_per_step": round(t1 * 1e3, 1),
                              "cores": 1},
            "sample": f"full workload convolve_apr (explicit pyramid of the same restricted levels), median of "
                      f"{len(times)} after a discarded cold run; single_thread: one run with threads = 1"}


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference (oracle/_ref, compiled from
    /root/reference's own headers) on the same workload.  Its input is made by
    the C restatement of generate_spheres + build_apr (oracle/build_oracle.c,
    bit-identical to the reference build; multi-threaded so it takes seconds,
    not the reference's 3 minutes / 34 GB) -- this process never loads the
    product library.  Then everything is the reference's own code:
    init_tree_structure, fill_tree, gaussian_stencil, make_pyramid, and the
    timed convolve_apr (all host threads)."""
    from pyoracle import Oracle, Ref, ref_available
    if args.config not in SPHERES:
        return {"impl": "reference", "unavailable": f"no host-side input for config {args.config} "
                                                    "(C4 is 548 M particles; the reference arm runs C1/C3)"}
    O = Oracle()
    n, count, rmin, rmax = SPHERES[args.config]
    t0 = time.time()
    leaf, values = O.build_spheres(n, count, rmin, rmax, blur=2.0, seed=42, rel_error=0.1)
    t_build = time.time() - t0
    n_pix = n ** 3
    k = args.stencil
    if not ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref (the compiled reference) is not on this box"}
    R = Ref()
    rapr = R.apr_from_arrays(leaf, (n, n, n))   # the reference's init_tree_structure
    k3, w = R.gaussian_stencil(1.0, k)
    t0 = time.time()
    rpyr = R.make_pyramid(w, k3, leaf.l_min, leaf.l_max, 0)   # PyramidMode::Restricted
    t_pyr = time.time() - t0
    threads = R.resolve_threads(0)
    tv = R.fill_tree(rapr, values, threads)
    n_p, n_t = leaf.particle_count(), int(tv.size)
    fn = lambda: R.convolve(rapr, values, tv, rpyr, 1, threads)  # noqa: E731
    fn()  # cold run discarded
    for _ in range(args.warmup):
        fn()
    times = []
    for _ in range(args.steps):
        a = time.perf_counter()
        fn()
        times.append(time.perf_counter() - a)
    t = float(np.mean(times))
    v = round(4 * n_pix / t / 1e9, 4)
    return {"metric": METRIC, "value": v, "unit": "GB/s (pixel-equivalent)", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 values, f64 accumulate", "data": "synthetic", "impl": "reference",
            "config": bench_config(args.config, k, n_p, n_t, n_pix),
            "input": "oracle/build_oracle.c (C restatement of generate_spheres + build_apr, bit-identical to the "
                     f"reference build; {t_build:.1f} s), make_pyramid {t_pyr:.1f} s",
            "parallelism": f"{threads} host threads",
            "particles_per_s": round(n_p / t, 1),
            "cpu_baseline": {"value": v, "unit": "GB/s (pixel-equivalent)", "cores": threads, "kind": "reference",
                             "sample": "full workload convolve_apr per step (unmodified reference, oracle/_ref)"},
            "e2e": {"value": v, "unit": "GB/s (pixel-equivalent)", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


DIMS = {"c1": (256, 256, 256), "c3": (1024, 1024, 1024), "c4": (4096, 4096, 2048)}


def write_bench_csv(path: str, res: dict, args) -> None:
    """Appends the result as rows of the reference's bench CSV schema
    (write_bench_csv, bench.hpp:33-42): image_id, dims, cr, op, stencil_size,
    wall_time_s, effective_throughput_Bps (4 bytes per pixel / time,
    metrics.hpp:15-21), memory_bytes_apr (particle in/out + interior values +
    the u16 y indices; the row arrays are not counted), memory_bytes_pixels
    (in + out), threads (host threads for CPU rows; 0 for GPU rows).  The op
    names the protocol: conv_apr (conv-only, device-resident), conv_apr_e2e
    (host buffers), conv_apr_paper (index + tree + conv), conv_pixels."""
    cfg = res.get("config", {})
    n_pix, n_p, n_t = cfg.get("pixels", 0), cfg.get("particles", 0), cfg.get("interior_nodes", 0)
    dims = "x".join(str(d) for d in DIMS.get(args.config, (0, 0, 0)))
    mem_apr, mem_pix = 8 * n_p + 4 * n_t + 2 * (n_p + n_t), 8 * n_pix
    rows = []

    def row(image, op, k, t_s, threads):
        if t_s and t_s > 0:
            rows.append(f"{image},{dims},{cfg.get('cr', 0)},{op},{k},{t_s:.9g},{4 * n_pix / t_s:.6g},{mem_apr},{mem_pix},"
                        f"{threads}")

    img = f"{args.config.upper()}"
    k = args.stencil
    if res.get("impl") == "reference":
        cb = res.get("cpu_baseline") or {}
        row(img + "/reference", "conv_apr", k, res.get("ms_per_step", 0) / 1e3, cb.get("cores", 0))
    else:
        row(f"{img}/{args.accum}", "conv_apr", k, res.get("ms_per_step", 0) / 1e3, 0)
        for name, v in (res.get("variants") or {}).items():
            kk, acc = name.split("_")
            row(f"{img}/{acc}", "conv_apr", int(kk[1:]), v.get("ms_per_step", 0) / 1e3, 0)
        e2e = res.get("e2e") or {}
        row(f"{img}/{args.accum}", "conv_apr_e2e", k, e2e.get("ms_per_step", 0) / 1e3, 0)
        pp = res.get("paper_protocol") or {}
        row(f"{img}/{args.accum}", "conv_apr_paper", k, pp.get("ms_per_step", 0) / 1e3, 0)
        px = res.get("convolve_pixels") or {}
        row(f"{img}/{args.accum}", "conv_pixels", k, px.get("ms", 0) / 1e3, 0)
        cb = res.get("cpu_baseline") or {}
        if cb.get("ms_per_step"):
            row(img + "/reference", "conv_apr", k, cb["ms_per_step"] / 1e3, cb.get("cores", 0))
            st = cb.get("single_thread") or {}
            row(img + "/reference", "conv_apr", k, st.get("ms_per_step", 0) / 1e3, st.get("cores", 0))
    new = not os.path.exists(path)
    with open(path, "a") as f:
        if new:
            f.write("image_id,dims,cr,op,stencil_size,wall_time_s,effective_throughput_Bps,memory_bytes_apr,"
                    "memory_bytes_pixels,threads\n")
        for r in rows:
            f.write(r + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=os.environ.get("APR_BENCH_CONFIG", "c3"), choices=["c1", "c3", "c4"])
    ap.add_argument("--stencil", type=int, default=3)
    ap.add_argument("--accum", default="exact", choices=["exact", "fast"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rl-iters", type=int, default=10)
    ap.add_argument("--csv", default=None, help="also append the result to this CSV (bench.hpp:33-42 schema)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        res = run_reference(args, rank, world)
        print(json.dumps(res), flush=True)
        if args.csv:
            write_bench_csv(args.csv, res, args)
        return
    # APRGPU_BENCH_SLAB=1 runs the N > 1 path (NCCL, z-slabs) with whatever world
    # size torchrun gives, 1 included: how the slab path is exercised on one GPU
    slab = world > 1 or os.environ.get("APRGPU_BENCH_SLAB") == "1"
    if slab:
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl")
    res = run_slab(args, rank, world) if slab else run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)
        if args.csv:
            write_bench_csv(args.csv, res, args)
    if slab:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

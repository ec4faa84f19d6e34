"""Benchmark: dual cells/s and iso triangles/s of the full hot path on the
626M-cell C4 soup (BASELINE.json configs[3], the configuration the metric is
quoted on; it fits one B200).

One step = the reference's build_index + extract_isosurface passes 1+2 on
one batch of synthetic input: pack (i,j,k,level) into 64-bit keys, radix
sort, gather scalars, build the search directory, then the fused dual
enumeration + ownership rules + marching cubes + ordered emission kernel.
`value` times that step with the unsorted cell soup already resident in HBM;
`e2e` times the same public call with pinned HOST input and output buffers
(H2D of 24 B/cell and D2H of the 72 B/triangle soup inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl amrx|reference]

Multi-GPU (torchrun, one rank per GPU, NCCL): rank 0 builds the index, the
sorted keys + scalars are broadcast over NVLink, every rank adopts them and
extracts its contiguous cell range; an all-gather of per-rank triangle
counts gives global output offsets.  Strong scaling: the 626M cells are
fixed, per-rank work shrinks with N.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref, the unmodified amriso sources) on a bounded sample of the same
workload with all host threads.
"""
from __future__ import annotations

import argparse
import gc
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

METRIC = "dual cells/sec & iso triangles/sec (626M-cell synthetic AMR), 1/2/4/8 B200"
HBM_FALLBACK = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region"""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def snapshot(self):
        """one sample right after a timed region too short for the 100 ms
        sampling interval"""
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=20).stdout
            self.lines += [ln.strip() for ln in out.splitlines() if ln.strip()]
            self.snapshot_only = True
        except Exception:
            pass

    def summary(self):
        if not self.lines:
            self.snapshot()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if getattr(self, "snapshot_only", False):
            out["note"] = "timed region shorter than the 100 ms sampling interval: one sample taken right after it"
        return out


# ---------------------------------------------------------------- workload
DATA_DESC = {
    "c1": "synthetic (reference generator gen_octree, sphere field)",
    "c2": "synthetic (reference generator random_slot_dataset, white noise)",
    "c3": "synthetic (GPU generator: 6-level octree toward a turbulent-noise zero set, soup order)",
    "c4": "synthetic (GPU generator: vortex-tube brick AMR, bijective-hash soup order)",
    "c5": "synthetic (GPU generator: brick AMR, generator order)",
    "deep": "synthetic (GPU generator: 13-level octree toward a landing-gear surface, 2-cell level bands, soup order)",
    "deep_thin": "synthetic (GPU generator: 13-level octree toward a landing-gear surface, 1-cell level bands, soup order)",
}


def make_workload(cfg_name, device):
    """device-resident synthetic input: (cells int32[n,4], scalars f64[n]) torch CUDA"""
    from paper_2004_08475_b200 import synth
    cfg = synth.CONFIGS[cfg_name]
    if cfg["kind"] == "bricks":
        b3 = cfg["bricks"]
        ds = synth.bricks(b3, seed=cfg["seed"], shuffle=cfg["shuffle"],
                          knobs=cfg.get("knobs", synth.C4_KNOBS), holes=synth.body_holes(b3))
        return ds.cells, ds.scalars, dict(bricks=list(b3), level_cells=ds.level_cells)
    import torch
    gen = getattr(synth, cfg["kind"])
    if cfg["kind"] in ("octree_noise", "octree_sdf"):  # GPU generators: device tensors
        cells, scal = gen(*cfg["args"], device=device, **cfg.get("kwargs", {}))
        return cells, scal, dict(level_cells=torch.bincount(cells[:, 3].long()).tolist())
    cells, scal = gen(*cfg["args"])
    return (torch.from_numpy(cells).to(device), torch.from_numpy(scal).to(device), {})


def iso_of(cfg_name):
    from paper_2004_08475_b200 import synth
    iso = synth.CONFIGS[cfg_name]["iso"]
    return synth.C4_ISO if iso is None else iso


# ---------------------------------------------------------------- amrx arm
def run_amrx(args):
    import torch
    import torch.distributed as dist
    import paper_2004_08475_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_dist:
        if "WORLD_SIZE" not in os.environ:  # --force-dist without a launcher: one rank
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
                              MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    iso = iso_of(args.config)

    # every rank generates the same input deterministically (the "batch")
    cells, scal, meta = make_workload(args.config, dev)
    n = cells.shape[0]
    n_levels = int(torch.unique(cells[:, 3]).numel())
    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    # output buffer sized from a first (untimed) run -- the process's first
    # calls, timed as the cold first call (library load, context, pool growth,
    # first-touch of every workspace; rounds make the extraction itself the
    # same work as a warm one)
    torch.cuda.synchronize()
    t_cold = time.perf_counter()
    idx = P.build_index(cells, scal, device=local, stream=sh, lookup=args.lookup)
    cold_build_ms = 1000 * (time.perf_counter() - t_cold)
    from paper_2004_08475_b200 import synth as S
    dual_only = bool(S.CONFIGS[args.config].get("dual_only"))
    if dual_only:  # C5: the dual mesh only (8 x u32 corners + u64 task id per dual)
        t_cold = time.perf_counter()
        dprobe = P.extract_dual_mesh(idx)
        cold_extract_ms = 1000 * (time.perf_counter() - t_cold)
        duals_full, ntri_full = len(dprobe.corners), 0
        del dprobe
        dcap = int(duals_full * 1.02) + 1024
        out_c = torch.empty((dcap, 8), dtype=torch.int32, device=dev)
        out_t = torch.empty(dcap, dtype=torch.int64, device=dev)
        out = torch.empty((1, 9), dtype=torch.float64, device=dev)
        cap = 1
    else:
        t_cold = time.perf_counter()
        probe = P.extract_isosurface(idx, P.IsoParams(iso=iso))
        cold_extract_ms = 1000 * (time.perf_counter() - t_cold)
        ntri_full = len(probe.fat)
        duals_full = probe.stats.duals_accepted
        del probe
        cap = int(ntri_full * 1.05) + 1024
        out = torch.empty((cap, 9), dtype=torch.float64, device=dev)
    geometry = idx.geometry()
    index_info = {"lookup": idx.info.lookup, "key_bits": idx.info.key_bits,
                  "lookup_entries": idx.info.lookup_entries, "max_probe": idx.info.max_probe,
                  "index_device_bytes": idx.info.device_bytes}
    idx.close()

    def step_single():
        ix = P.build_index(cells, scal, device=local, stream=sh, lookup=args.lookup)
        if dual_only:
            d = P.extract_dual_mesh(ix, out=(out_c, out_t))
            ingest = ix.info.seconds_ingest
            ix.close()
            return d.stats, ingest, 0
        r = P.extract_isosurface(ix, P.IsoParams(iso=iso), out=out)
        ingest = ix.info.seconds_ingest
        ix.close()
        return r.stats, ingest, len(r.fat)

    from paper_2004_08475_b200 import dist as D

    # each rank holds a slice of the (shuffled) cell list
    lo_c, hi_c = n * rank // max(world, 1), n * (rank + 1) // max(world, 1)
    my_cells, my_scal = cells[lo_c:hi_c], scal[lo_c:hi_c]

    def step_multi():
        if args.dist_mode == "replicate":
            # rank 0 sorts; NCCL broadcast of the sorted keys + scalars; each
            # rank adopts them and extracts its own contiguous cell range
            ix = D.replicate_index(cells if rank == 0 else None,
                                   scal if rank == 0 else None, device=dev, stream=sh)
            ingest = ix.info.seconds_ingest
            res = D.extract_isosurface_partitioned(ix, P.IsoParams(iso=iso), out=out,
                                                   device=dev)
            ix.close()
            return res.stats, ingest, res.total
        # distributed build: slice sort, sampled splitters, all-to-all by
        # key range (+ halo), partition index; owned-range extraction; an
        # all-gather of per-rank counts gives the global offsets
        di = D.build_distributed(my_cells, my_scal, device=dev, stream=sh)
        ingest = di.index.info.seconds_ingest if di.index is not None else 0.0
        res = D.extract_isosurface_distributed(di, P.IsoParams(iso=iso), out=out, device=dev)
        if di.index is not None:
            di.index.close()
        return res.stats, ingest, res.total

    step = step_multi if (world > 1 or args.force_dist) else step_single
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    launches0 = P.kernel_launches()
    kernel_s, ingest_s, tris = [], [], 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st, ing, nt = step()
            kernel_s.append(st.seconds_pass1)
            ingest_s.append(ing)
            tris = nt
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - t0
    launches = P.kernel_launches() - launches0
    # the library syncs its stream per call, so the events on that stream
    # bracket every step; host-side gaps between calls are included
    ms_dev = ev0.elapsed_time(ev1) / args.steps
    ms = max(ms_dev, 1000.0 * wall / args.steps)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())

    # ---- e2e through the same public call with pinned host buffers
    e2e = None
    if world > 1 and not args.no_e2e:
        # every rank's slice from pinned host memory, its part of the soup
        # into pinned host memory
        hcells = torch.empty(my_cells.shape, dtype=torch.int32, pin_memory=True)
        hscal = torch.empty(my_scal.shape, dtype=torch.float64, pin_memory=True)
        hcells.copy_(my_cells)
        hscal.copy_(my_scal)
        hout = torch.empty((int(cap * 1.5 / world) + 4096, 9), dtype=torch.float64,
                           pin_memory=True)

        def step_e2e_multi():
            di = D.build_distributed(hcells, hscal, device=dev, stream=sh)
            res = D.extract_isosurface_distributed(di, P.IsoParams(iso=iso), out=hout,
                                                   device=dev)
            if di.index is not None:
                di.index.close()
            return res.total, len(res.fat)

        step_e2e_multi()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        k2 = max(1, min(args.steps, 3))
        mine = 0
        for _ in range(k2):
            nt, mine = step_e2e_multi()
        torch.cuda.synchronize()
        dist.barrier()
        ms_e2e = 1000 * (time.perf_counter() - t0) / k2
        mt = torch.tensor([ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms_e2e = float(mt.item())
        e2e = {"value": duals_full / (ms_e2e / 1000.0), "unit": "dual cells/s",
               "ms_per_step": ms_e2e, "triangles_per_s": nt / (ms_e2e / 1000.0),
               "h2d_bytes_per_step": int(n * 24), "d2h_bytes_per_step": int(nt * 72),
               "note": "every rank uploads its slice and downloads its part; bytes are job totals"}
        del hcells, hscal, hout
    # the weld (not part of the step: the reference arm excludes it too),
    # once on the device-resident soup of the last step
    weld_ms = None
    if world == 1 and not dual_only:
        wsoup = out[:tris]
        P.weld(wsoup)  # warm-up (the pool grows to the weld's buffers once)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mesh = P.weld(wsoup)
        torch.cuda.synchronize()
        weld_ms = 1000 * (time.perf_counter() - t0)
        weld_info = {"ms": weld_ms, "triangles": int(tris), "vertices": len(mesh.vertices),
                     "note": "amrx_weld, device soup -> device indexed mesh"}
        del mesh

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    hbm, kind = peaks()
    kern_ms = 1000.0 * statistics.mean(kernel_s)
    # algorithmic bytes: iso 16 B/cell + 72 B/triangle; dual
    # mesh 8 B/cell + 40 B/dual (corners + task id)
    alg_bytes = (n * 8 + duals_full * 40) / world if dual_only else \
        n * 16 / world + tris * 72 / world
    achieved = alg_bytes / (kern_ms / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config)
        except Exception:
            traffic = None
    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(cells, scal, iso, args)
    if world == 1 and not args.no_e2e and not dual_only:
        # pinned host copies of the input; the device copies, the device
        # soup and the step's tensors go back to the pool first (the
        # pipelined e2e holds two indexes at a time)
        hcells = torch.empty(cells.shape, dtype=torch.int32, pin_memory=True)
        hscal = torch.empty(scal.shape, dtype=torch.float64, pin_memory=True)
        hcells.copy_(cells)
        hscal.copy_(scal)
        del cells, scal, out, my_cells, my_scal
        torch.cuda.empty_cache()
        P.release_cached_memory()
        e2e = e2e_single(P, hcells, hscal, iso, cap, duals_full, n, local, sh, args)
        if not args.e2e_single_only:
            try:
                pipe = e2e_pipelined(P, hcells, hscal, iso, cap, n, local, sh, args)
            except Exception as exc:  # device memory: keep the single-step line
                pipe = {"error": f"{type(exc).__name__}: {exc}"[:200]}
            e2e["pipelined"] = pipe
            if "ms_per_step" in pipe and pipe["ms_per_step"] < e2e["ms_per_step"]:
                # the headline e2e is the steady state of consecutive steps
                e2e["single_step"] = {k: e2e[k] for k in ("value", "ms_per_step",
                                                           "triangles_per_s")}
                e2e["value"] = duals_full / (pipe["ms_per_step"] / 1000.0)
                e2e["triangles_per_s"] = pipe["triangles"] / (pipe["ms_per_step"] / 1000.0)
                e2e["ms_per_step"] = pipe["ms_per_step"]
                e2e["steps"] = pipe["steps"]
                e2e["mode"] = ("steady state of consecutive steps: build_index from the pinned "
                               "host input, extract_isosurface into a device soup, its download "
                               "overlapping the next step's upload (full-duplex host link); "
                               "every step's H2D and D2H in the timed region, the timer stops "
                               "after the last download; single_step = one step alone with a "
                               "pinned host soup")
        del hcells, hscal

    line = {
        "metric": METRIC,
        "value": duals_full / (ms / 1000.0),
        "unit": "dual cells/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "int64 keys / f64 scalars",
        "data": DATA_DESC.get(args.config, "synthetic"),
        "config": {"workload": f"{args.config}: {n} cells, {n_levels} levels, " +
                               ("dual mesh only" if dual_only else f"iso {iso}"),
                   "cells": n, "triangles": tris, "duals": duals_full, "iso": iso,
                   "parallelism": (f"distributed sort + range partition x{world}" if args.dist_mode == "partition" else f"rank-0 sort + broadcast x{world}") if world > 1 else "single GPU",
                   "l2": "inputs (24 B/cell) far larger than L2", "index": index_info, **meta},
        "iso_triangles_per_s": tris / (ms / 1000.0),
        "paper_split_ms": {"X_extract_kernel": kern_ms, "ingest_sort": 1000 * statistics.mean(ingest_s),
                           "Y_step": ms},
        "cold_first_call_ms": {"build_index": cold_build_ms, "extract": cold_extract_ms,
                               "note": "the process's first calls (host output, wall clock), "
                                       "beside the warm device step"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": ("dual mesh: extract_kernel<dual>" if dual_only else
                                "iso extraction: extract_kernel<iso, f64> + mc_jobs_kernel<f64> "
                                "(CUDA events around both launches)"), "peak_kind": kind,
                     "alg_bytes_per_launch": alg_bytes,
                     "note": ("not bandwidth bound: extract_kernel issues instructions on "
                              "78% of cycles at 4% of DRAM peak; mc_jobs_kernel waits on "
                              "the corner-scalar loads (long scoreboard) at 26% of DRAM peak "
                              "(profiles/r02_extract_c4_ncu.txt)")},
        "weld": weld_info if weld_ms is not None else None,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    if dist.is_initialized():
        dist.destroy_process_group()


def link_times(hcells, hscal, hout, dev):
    """the host link alone: the e2e step's upload (cells + scalars) and
    download (the soup) as plain pinned copies, timed with CUDA events --
    the floor the e2e number is measured against"""
    import torch
    dc = torch.empty(hcells.shape, dtype=hcells.dtype, device=dev)
    ds = torch.empty(hscal.shape, dtype=hscal.dtype, device=dev)
    do = torch.empty(hout.shape, dtype=hout.dtype, device=dev)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dc.copy_(hcells, non_blocking=True)  # warm
    torch.cuda.synchronize()
    e[0].record()
    dc.copy_(hcells, non_blocking=True)
    ds.copy_(hscal, non_blocking=True)
    e[1].record()
    e[2].record()
    hout.copy_(do, non_blocking=True)
    e[3].record()
    torch.cuda.synchronize()
    up, down = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])
    nb_up = hcells.numel() * hcells.element_size() + hscal.numel() * hscal.element_size()
    nb_down = hout.numel() * hout.element_size()
    return {"h2d_ms": up, "d2h_ms": down, "h2d_gbs": nb_up / up / 1e6 if up else None,
            "d2h_gbs": nb_down / down / 1e6 if down else None,
            "note": "pinned copies of the step's bytes alone (the host-link floor of e2e)"}


def e2e_single(P, hcells, hscal, iso, cap, duals_full, n, local, sh, args):
    """e2e on one GPU through the public calls (build_index +
    extract_isosurface) from pinned host input to a pinned host soup, every
    step's H2D and D2H inside the timed region.  (Overlapping consecutive
    steps -- step i+1's upload + sort beside step i's extraction + download
    -- was measured slower, 963 vs 467 ms per C4 step: DESIGN.md §7.)"""
    import torch
    hout = torch.empty((cap, 9), dtype=torch.float64, pin_memory=True)

    def step_e2e():
        ix = P.build_index(hcells, hscal, device=local, stream=sh, lookup=args.lookup)
        r = P.extract_isosurface(ix, P.IsoParams(iso=iso), out=hout)
        ix.close()
        return len(r.fat)

    for _ in range(2):
        step_e2e()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(sh) if sh else torch.cuda.current_stream()
    gc.collect()
    gc.disable()  # no collector pause inside the wall-clock region
    e0.record(stream)
    t0 = time.perf_counter()
    k2 = max(1, min(args.steps, 3))
    for _ in range(k2):
        nt = step_e2e()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max(e0.elapsed_time(e1) / k2, 1000 * (time.perf_counter() - t0) / k2)
    gc.enable()
    link = link_times(hcells, hscal, hout[:nt], torch.device("cuda", local))
    del hout
    return {"value": duals_full / (ms_e2e / 1000.0), "unit": "dual cells/s",
            "ms_per_step": ms_e2e, "triangles_per_s": nt / (ms_e2e / 1000.0),
            "h2d_bytes_per_step": int(n * 16 + n * 8), "d2h_bytes_per_step": int(nt * 72),
            "steps": k2, "link": link}


def e2e_pipelined(P, hcells, hscal, iso, cap, n, local, sh, args, keep=False):
    """steady-state e2e of consecutive steps through the same public calls:
    build_index from pinned host input, extract_isosurface into one of two
    device soups, then that soup's download on a side stream -- which runs
    while the next step uploads its input (the host link is full duplex).
    Every step's H2D (24 B/cell) and D2H (72 B/triangle) is inside the timed
    region; the timer stops after the last download."""
    import torch
    dev = torch.device("cuda", local)
    hout = torch.empty((cap, 9), dtype=torch.float64, pin_memory=True)
    dsoup = [torch.empty((cap, 9), dtype=torch.float64, device=dev) for _ in range(2)]
    main = torch.cuda.ExternalStream(sh, device=dev) if sh else torch.cuda.current_stream(dev)
    down = torch.cuda.Stream(device=dev)
    done = [None, None]

    def step(i):
        b = i & 1
        if done[b] is not None:  # the soup buffer's previous download (long done by now)
            done[b].synchronize()
        ix = P.build_index(hcells, hscal, device=local, stream=sh, lookup=args.lookup)
        r = P.extract_isosurface(ix, P.IsoParams(iso=iso), out=dsoup[b])
        ix.close()
        nt = len(r.fat)
        ev = torch.cuda.Event()
        ev.record(main)
        down.wait_event(ev)
        with torch.cuda.stream(down):
            hout[:nt].copy_(dsoup[b][:nt], non_blocking=True)
            done[b] = torch.cuda.Event()
            done[b].record(down)
        return nt

    step(0)
    step(1)
    torch.cuda.synchronize(dev)
    k2 = max(2, min(args.steps, 8))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()  # no collector pause inside the wall-clock region
    e0.record(main)
    t0 = time.perf_counter()
    for i in range(k2):
        nt = step(i)
    main.wait_stream(down)
    e1.record(main)
    torch.cuda.synchronize(dev)
    ms = max(e0.elapsed_time(e1) / k2, 1000 * (time.perf_counter() - t0) / k2)
    gc.enable()
    res = {"ms_per_step": ms, "steps": k2, "triangles": nt,
           "h2d_bytes_per_step": int(n * 24), "d2h_bytes_per_step": int(nt * 72)}
    if keep:  # tests: the last step's downloaded soup
        res["_soup"] = hout[:nt].clone()
    del hout, dsoup
    return res


# ------------------------------------------------------------ CPU baseline
def cpu_sample(cells, scal, target):
    """a contiguous sub-box (x slabs) of the workload with ~target cells"""
    import torch
    x = cells[:, 0]
    xs = torch.sort(x).values
    n = len(xs)
    lo = int(xs[n // 3].item())
    # grow the slab range until it holds ~target cells
    hi_idx = min(n - 1, n // 3 + target)
    hi = int(xs[hi_idx].item())
    m = (x >= lo) & (x < hi)
    return cells[m].cpu().numpy(), scal[m].cpu().numpy(), (lo, hi)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cells, scal, iso, args, impl_line=False, t1=True):
    """the reference (oracle/_ref) on a bounded sample; reports dual cells/s
    over build_index (serial sort) + passes 1+2 (all host threads)"""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles
    R = oracles.reference()
    kind = "reference"
    if R is None:
        R = oracles.restatement()
        kind = "port"
    hc, hs, slab = cpu_sample(cells, scal, args.cpu_sample)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    h = R.build(hc, hs)
    t_build = time.perf_counter() - t0
    from paper_2004_08475_b200 import synth as S
    dual_only = bool(S.CONFIGS[args.config].get("dual_only"))
    if kind == "reference" and dual_only:
        R.extract_dual(h, threads)  # warm-up
        t1 = time.perf_counter()
        res = R.extract_dual(h, threads)
        t_ext = time.perf_counter() - t1
        duals = len(res["corners"])
        tris = 0
        weld = None
        cores = threads
    elif kind == "reference":
        # warm-up (first run per process is 2-7x slower)
        R.extract_iso(h, iso, threads)
        res = R.extract_iso(h, iso, threads)
        st = res["stats"]
        t_ext = st["seconds_pass1"] + st["seconds_pass2"]
        duals = st["duals_accepted"]
        tris = st["fat_triangle_count"]
        weld = st["seconds_weld"]
        cores = threads
    else:
        t1 = time.perf_counter()
        r = R.extract_iso(h, iso)
        t_ext = time.perf_counter() - t1
        duals = int(r["counters"][0])
        tris = len(r["fat"])
        weld = None
        cores = 1
    R.free(h)
    total = t_build + t_ext
    out = {"value": duals / total, "unit": "dual cells/s", "cores": cores, "kind": kind,
           "sample": f"{len(hc)} cells (x-slabs [{slab[0]},{slab[1]}) of the workload), "
                     f"build_index {t_build:.2f} s (serial) + passes 1+2 {t_ext:.2f} s "
                     f"({cores} threads); weld excluded ({weld})",
           "triangles_per_s": tris / total, "seconds": total, "cpu_model": cpu_model(),
           "nproc": os.cpu_count()}
    if t1 and kind == "reference":
        # the reference at T=1 (parallel.hpp:33-42 thread count 1) on a
        # smaller slab of the same workload, ~10 s of CPU
        hc1, hs1, slab1 = cpu_sample(cells, scal, max(1, args.cpu_sample // 8))
        tb = time.perf_counter()
        h1 = R.build(hc1, hs1)
        tb = time.perf_counter() - tb
        if dual_only:
            R.extract_dual(h1, 1)
            t0 = time.perf_counter()
            d1 = len(R.extract_dual(h1, 1)["corners"])
            te = time.perf_counter() - t0
        else:
            R.extract_iso(h1, iso, 1)
            st1 = R.extract_iso(h1, iso, 1)["stats"]
            te = st1["seconds_pass1"] + st1["seconds_pass2"]
            d1 = st1["duals_accepted"]
        R.free(h1)
        out["t1"] = {"value": d1 / (tb + te), "unit": "dual cells/s", "cores": 1,
                     "sample": f"{len(hc1)} cells (x-slabs [{slab1[0]},{slab1[1]})), build_index "
                               f"{tb:.2f} s + passes 1+2 {te:.2f} s (1 thread)"}
    return out


def run_reference(args):
    """--impl reference: the reference CPU path on the same workload (rank 0)"""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    iso = iso_of(args.config)
    cells, scal, meta = make_workload(args.config, torch.device("cuda"))
    n = cells.shape[0]
    vals = []
    cb = None
    for _ in range(args.warmup):
        cpu_baseline(cells, scal, iso, args, t1=False)
    for _ in range(args.steps):
        cb = cpu_baseline(cells, scal, iso, args, t1=False)
        vals.append(cb["value"])
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "dual cells/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * cb["seconds"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32 cells / f64 scalars", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n} cells (bounded sample per step)", **meta},
        "cpu_baseline": {**cb, "value": v},
        "e2e": {"value": v, "unit": "dual cells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n, argv):
    """--gpus N without a launcher: re-run this script under torchrun with N
    ranks on this node (one per GPU), NCCL_DEBUG=INFO so the communicator
    lines show the rank count; returns the launcher's exit code"""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout carries the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def selftest(args):
    """--selftest: the multi-rank plumbing only (gloo on CPU): every rank
    joins, an all-reduce of the ranks and a max-over-ranks timing, rank 0
    prints one line -- what tests/test_bench_spawn.py runs"""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t)
    ms = torch.tensor([1.0 + rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"selftest": "ok", "n_gpus": world, "rank_sum": float(t.item()),
                          "ms_max": float(ms.item()),
                          "nccl_debug": os.environ.get("NCCL_DEBUG")}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amrx", choices=["amrx", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--cpu-sample", type=int, default=12_000_000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-single-only", action="store_true",
                    help="skip the steady-state (pipelined) e2e measurement")
    ap.add_argument("--dist-mode", default="partition", choices=["partition", "replicate"],
                    help="multi-GPU build: distributed sort + exchange, or rank-0 sort + broadcast")
    ap.add_argument("--lookup", default=None, choices=["records", "hash", "directory"],
                    help="force the index lookup structure (default: chosen from the key space)")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU code path even at world size 1 (testing)")
    ap.add_argument("--selftest", action="store_true",
                    help="multi-rank plumbing check over gloo (no GPU work)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus, sys.argv[1:]))
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.selftest:
        selftest(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_amrx(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — Hierarchy-Scan + fused Bind MeshPose throughput on B200.

Metric (BASELINE.json): joints/s of Hierarchy-Scan + skin, with HBM GB/s against
the measured peak.  Default workload: config 5 — 1,000,000 mixed characters
(333,334 hum64 + 333,333 chain256 + 333,333 tree1024; 448 M joints, 64.5 GB of
algorithmic HBM traffic per step) per GPU (weak scaling: rank r owns global
characters [r*1M, (r+1)*1M) of an N-million crowd; no collective on the path).

A step = one hs_scan per skeleton type over that rank's characters (3 launches),
inputs resident in HBM (21.5 GB of local poses, larger than the 126 MB L2, so no
flush is needed).  Launch (N > 1):
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P bench.py --gpus N
``--impl reference`` times the fp64 CPU oracle (the reference arm of this tier)
on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import hsgen  # noqa: E402

BYTES_PER_JOINT = 144  # 48 local in + 48 global out + 48 skin out
# --stage1: the algorithmic minimum is 96 B per joint (+16 B per layer per character): the
# local pose need not touch HBM (the fused placement); the default two-pass placement moves
# 192 B/joint but runs faster, and the roofline is taken against 96
STAGE1_BYTES_PER_JOINT = 96
STAGE1_CLIPS, STAGE1_KEYS, STAGE1_FPS, STAGE1_LAYERS, STAGE1_SPAN = 8, 31, 30.0, 2, 1.5
METRIC = "joints/sec (Hierarchy-Scan+skin) and HBM GB/s vs peak at 1/2/4/8 B200"
WORKLOAD_NAME = {1: "C1 1,000 x hum32 (L=8)", 2: "C2 100,000 x hum64 (L=12)",
                 3: "C3 50,000 x chain256 (L=256)", 4: "C4 20,000 x tree1024 (L=300)",
                 5: "C5 1,000,000 mixed hum64/chain256/tree1024 per GPU",
                 6: "C6 2,000 x tree16384 (L=1024, beyond one CTA: multi-tile path)",
                 7: "C7 2,000 x tree16384, depth-first labels (multi-tile path)"}


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5, 6, 7])
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--cpu-frac", type=int, default=8,
                    help="cpu_baseline / reference sample = n_chars // this, per skeleton type")
    ap.add_argument("--e2e-frac", type=int, default=8,
                    help="e2e host-buffer slice = n_chars // this, per skeleton type")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--algo", default="auto", help="hs_scan_ex algorithm (comparisons)")
    ap.add_argument("--tile-ctas", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--tile-joints", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--sbufs", type=int, default=0)
    ap.add_argument("--pbuf", type=int, default=0)
    ap.add_argument("--chunking", type=int, default=0, help="1 = consecutive, 2 = heavy-path pieces")
    ap.add_argument("--stage1", action="store_true",
                    help="fused Stage-1 prologue (hs_animate): 2 animation layers per character "
                         "sampled from 8 clips x 31 keys instead of resident local poses")
    ap.add_argument("--skin-mesh", type=int, default=0, metavar="V",
                    help="NEXT-4: fuse linear blend skinning of a V-vertex synthetic mesh per "
                         "character (hs_scan_skin); 0 = off")
    ap.add_argument("--launch", choices=["auto", "batch", "per-type"], default="auto",
                    help="batch = all skeleton types in one hs_scan_batch launch (NEXT-3); "
                         "auto = batch for small crowds only (see bench.py)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no checks, no e2e, no cpu baseline")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N > 1 (gloo: CPU collectives, lets a test run "
                         "several ranks on one GPU; the data path has no collective either way)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config single-type launches (C2, C3, C4, C6, C7) reported in "
                         "the line's 'configs' object")
    ap.add_argument("--no-validate", action="store_true",
                    help="skip the N > 1 validation (all-gather of sampled G/S shards, bitwise "
                         "check against a single-rank recomputation)")
    return ap.parse_args(argv)


# ------------------------------------------------------------------------ helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def shard(n_total: int, rank: int, world: int, scaling: str):
    """(global first character, count) of this rank's characters for one skeleton type."""
    if scaling == "weak":
        return rank * n_total, n_total
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def coll_device(backend: str, device):
    """Tensors for collectives: CPU under gloo, the rank's GPU under NCCL."""
    return "cpu" if backend == "gloo" else device


def reduce_over_ranks(ms_rank: float, joints_rank: int, world: int, device):
    """(max over ranks of the timed-region ms, sum over ranks of joints processed).
    Outside the timed region; NCCL on the GPU path, gloo in the CPU tests."""
    if world <= 1:
        return ms_rank, joints_rank
    import torch
    import torch.distributed as dist
    mx = torch.tensor([ms_rank], dtype=torch.float64, device=device)
    sm = torch.tensor([float(joints_rank)], dtype=torch.float64, device=device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx.item()), int(sm.item())


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ best of 10)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(workload: str, kernel: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full summary,
    only when it was captured on this workload and launch AND on these exact library
    sources (the capture records their hash; any source change makes it stale -> null)."""
    import paper_2505_06703_b200 as hs
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        entries = json.load(open(path))
        entries = entries if isinstance(entries, list) else [entries]
    except Exception:
        return None, "no profiles/ncu_traffic.json"
    sha = hs.sources_sha256()
    for d in entries:
        if d.get("workload") == workload and d.get("kernel") == kernel:
            if d.get("sources_sha256") != sha:
                return None, f"stale capture ({d.get('source')}: sources {d.get('sources_sha256')} != {sha})"
            return float(d["dram_bytes_per_launch"]), d.get("source")
    return None, "no capture for this workload / kernel"


class ClockSampler:
    """NVML SM-clock and clock-event-reason samples while running (every 20 ms)."""

    REASONS = [("gpu_idle", 0x1), ("applications_clocks_setting", 0x2), ("sw_power_cap", 0x4),
               ("hw_slowdown", 0x8), ("sync_boost", 0x10), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80),
               ("display_clock_setting", 0x100)]

    def __init__(self, index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        names = [n for n, bit in self.REASONS if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------ reference arm
def run_reference(args):
    """The tier's reference arm: the fp64 CPU oracle as it stands, on host cores."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    types = hsgen.CONFIGS[args.config]
    sample = []
    for name, n, seed, type_, ib_seed in types:
        par = hsgen.skeleton(name)
        m = max(1, n // args.cpu_frac)
        sample.append((name, par, hsgen.local_poses(seed, len(par), m, type_=type_),
                       hsgen.inv_bind(ib_seed, len(par))))
    joints = sum(len(p) * loc.shape[0] for _, p, loc, _ in sample)
    cores = host_cores()

    def step():
        for _, par, loc, ib in sample:
            oracle.scan_discard(par, loc, ib, nthreads=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = joints * args.steps / dt
    desc = ", ".join(f"{loc.shape[0]} x {name}" for name, _, loc, _ in sample)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "joints/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD_NAME[args.config] + f" (1/{args.cpu_frac} sample)",
                       "sample": desc, "joints_per_step": joints},
            "cpu_baseline": {"value": value, "unit": "joints/s", "cores": cores, "kind": "oracle",
                             "sample": desc, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "joints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line, args)
    return 0


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "a") as f:
            f.write(s + "\n")


# ------------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2505_06703_b200 as hs

    rank, local_rank, world = dist_env()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    # one process per GPU; a gloo test may run several ranks on one GPU (no collective
    # on the data path, so ranks never wait on each other's kernels)
    gpu = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group("gloo")
    hs.lib()  # fails loudly when libhs.so is missing: no fallback path exists
    hsgen.lib_cuda()
    dev = torch.device("cuda", gpu)
    cdev = coll_device(args.dist_backend, dev)
    stream = torch.cuda.current_stream()

    # ---- workload: one skeleton handle and one resident crowd per skeleton type
    work = []
    for name, n_total, seed, type_, ib_seed in hsgen.CONFIGS[args.config]:
        par = hsgen.skeleton(name)
        J = len(par)
        ib = hsgen.inv_bind(ib_seed, J)
        c0, n = shard(n_total, rank, world, args.scaling)
        sk = hs.Skeleton(par, ib, chunk=args.chunk, tile_joints=args.tile_joints,
                         stages=args.stages, sbufs=args.sbufs, pbuf=args.pbuf,
                         chunking=args.chunking)
        item = dict(name=name, par=par, ib=ib, J=J, c0=c0, n=n, seed=seed, type=type_, sk=sk)
        if args.stage1:
            keys = hsgen.clips(100 + type_, J, STAGE1_CLIPS, STAGE1_KEYS, type_=type_)
            item["keys"] = keys
            item["cs"] = hs.ClipSet(sk, keys, STAGE1_FPS, 1)
            lay = hsgen.layers(seed, n, STAGE1_LAYERS, STAGE1_CLIPS, STAGE1_SPAN, char0=c0, type_=type_)
            item["lay_np"] = lay
            item["layers"] = torch.from_numpy(lay.view(np.int32).reshape(n, STAGE1_LAYERS, 4)).to(dev)
            item["g"] = torch.empty((n, J, 3, 4), dtype=torch.float32, device=dev)
            if args.skin_mesh:   # the whole pipeline: Stage 1 -> scan -> bind -> skinning
                item["mesh_np"] = hsgen.mesh(200 + type_, par, args.skin_mesh, type_=type_)
                item["mesh"] = hs.Mesh(sk, *item["mesh_np"])
                item["verts"] = torch.empty((n, args.skin_mesh, 3), dtype=torch.float32, device=dev)
        else:
            local = torch.empty((n, J, 3, 4), dtype=torch.float32, device=dev)
            if n:
                rc = hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, c0, n, local.data_ptr(),
                                                           stream.cuda_stream)
                assert rc == 0, f"generator launch failed: {rc}"
            item["local"] = local
            item["g"] = torch.empty_like(local)
            if args.skin_mesh:
                item["mesh_np"] = hsgen.mesh(200 + type_, par, args.skin_mesh, type_=type_)
                item["mesh"] = hs.Mesh(sk, *item["mesh_np"])
                item["verts"] = torch.empty((n, args.skin_mesh, 3), dtype=torch.float32, device=dev)
        item["s"] = torch.empty_like(item["g"])
        work.append(item)
    torch.cuda.synchronize()
    joints_rank = sum(w["n"] * w["J"] for w in work)

    # auto: one batch launch only when every type's crowd is small (under ~32 tiles per
    # SM, where per-launch fill/drain and tails dominate; profiles/r01f_next3_sweep.json);
    # C5's crowds are thousands of tiles per SM, where per-type launches measured 3%
    # faster (the multi-segment kernel's program switch costs registers); a single type
    # runs hs_scan, whose small-crowd program keeps every SM busy
    small = all(-(-w["n"] // max(1, w["sk"].query("tile_chars"))) < 32 * 148 for w in work)
    batch = args.launch == "batch" or (
        args.launch == "auto" and small and len(work) > 1 and not args.stage1 and not args.skin_mesh and args.algo == "auto"
        and args.tile_ctas == 0 and len({w["sk"].query("chunk") for w in work}) == 1
        and all(w["sk"].query("path") == 1 for w in work))
    # launches per step: one hs_scan_batch over every type, or one call per type
    launches = [("batch", list(range(len(work))))] if batch else [(w["name"], [t]) for t, w in
                                                                   enumerate(work)]
    batch_items = [(w["sk"], w["local"], w["g"], w["s"]) for w in work if w["n"]] if batch else None

    def step(events=None, k=0):
        for li, (_, members) in enumerate(launches):
            if events is not None:
                events[li][0][k].record(stream)
            if batch:
                hs.scan_batch(batch_items, stream=stream)
            else:
                w = work[members[0]]
                if args.stage1 and args.skin_mesh:   # the whole pipeline in one call
                    hs.animate_skin(w["sk"], w["cs"], w["layers"], w["mesh"], w["g"], w["s"], w["verts"],
                                    stream=stream)
                elif args.stage1:
                    hs.animate(w["sk"], w["cs"], w["layers"], w["g"], w["s"], stream=stream)
                elif args.skin_mesh:
                    hs.scan_skin(w["sk"], w["mesh"], w["local"], w["g"], w["s"], w["verts"], stream=stream)
                else:
                    w["sk"].scan_into(w["local"], w["g"], w["s"], stream=stream, algo=args.algo,
                                      tile_ctas=args.tile_ctas)
            if events is not None:
                events[li][1][k].record(stream)

    # ---- correctness on sampled characters at full size (outside the timed region)
    step()
    torch.cuda.synchronize()
    check = None
    if not (args.no_check or args.profile):
        check = sampled_parity(work, rank)
        if world > 1:   # every rank checks its own shard; the job passes only if all do
            worst = torch.tensor([check["worst"]], dtype=torch.float64, device=cdev)
            dist.all_reduce(worst, op=dist.ReduceOp.MAX)
            check["worst_all_ranks"] = float(worst.item())
            check["pass"] = check["worst_all_ranks"] <= check["tolerance"]

    # ---- warm-up, then exactly K timed steps between barrier + synchronize
    for _ in range(args.warmup):
        step()
    K = args.steps
    events = [[[torch.cuda.Event(enable_timing=True) for _ in range(K)] for _ in range(2)]
              for _ in launches]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(torch.cuda.current_device())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        start.record(stream)
        for k in range(K):
            step(events, k)
        stop.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_rank = start.elapsed_time(stop)
    launch_ms = [[events[li][0][k].elapsed_time(events[li][1][k]) for k in range(K)]
                 for li in range(len(launches))]
    per_launch_ms = [statistics.mean(x) for x in launch_ms]
    ms, joints_total = reduce_over_ranks(ms_rank, joints_rank, world, cdev)
    value = joints_total * K / (ms / 1e3)

    # ---- roofline of the dominant kernel launch (largest byte share: the batch launch,
    # else tree1024's)
    bpj = STAGE1_BYTES_PER_JOINT if args.stage1 else BYTES_PER_JOINT
    per_char_extra = (16 * STAGE1_LAYERS if args.stage1 else 0) + 12 * args.skin_mesh

    def launch_bytes(li):
        return sum(bpj * work[t]["n"] * work[t]["J"] + per_char_extra * work[t]["n"]
                   for t in launches[li][1])

    dom_l = max(range(len(launches)), key=launch_bytes)
    dom = max(launches[dom_l][1], key=lambda t: work[t]["n"] * work[t]["J"])
    dom_bytes = launch_bytes(dom_l)
    achieved = dom_bytes / (per_launch_ms[dom_l] / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    workload = WORKLOAD_NAME[args.config]
    if args.skin_mesh:
        workload += f" + LBS ({args.skin_mesh}-vertex mesh per character)"
    if args.stage1:
        workload += (f" + Stage 1 ({STAGE1_LAYERS} layers per character, "
                     f"{STAGE1_CLIPS} clips x {STAGE1_KEYS} keys at {STAGE1_FPS:g} fps)")
    dom_two_pass_lbs = bool(args.skin_mesh) and args.skin_mesh >= 2 * work[dom]["J"]
    kernel_name = (f"stage1_kernel + chunked_kernel{'<lbs>' if args.skin_mesh else ''} (two-pass "
                   f"{'hs_animate_skin' if args.skin_mesh else 'hs_animate'}, {launches[dom_l][0]} call)"
                   if args.stage1 else
                   f"chunked_kernel + lbs_kernel (two-pass hs_scan_skin, {launches[dom_l][0]} call)"
                   if dom_two_pass_lbs else
                   f"seq_kernel (multi-tile path, {launches[dom_l][0]} launch)"
                   if work[dom]["sk"].query("path") == 7 and args.algo in ("auto", "tiles") else
                   f"chunked_kernel{'<lbs>' if args.skin_mesh else ''} ({launches[dom_l][0]} launch)")
    traffic, traffic_src = ncu_traffic(workload, kernel_name)

    # ---- the other configs' single-type launches (deep-skeleton and multi-tile targets,
    # driver-visible): after the timed region, each on its own resident inputs
    configs = None
    if (args.config == 5 and world == 1 and not (args.no_configs or args.profile or args.stage1
                                                  or args.skin_mesh or args.algo != "auto")):
        configs = measure_configs(hs, torch, stream, dev)
    # ---- N > 1: assemble sampled G/S shards from every rank (outside the timed region)
    # and check them bitwise against this rank's own recomputation of those characters
    validation = None
    if world > 1 and not (args.no_validate or args.profile or args.stage1 or args.skin_mesh):
        validation = validate_across_ranks(work, args, hs, torch, dist, rank, world, dev, cdev)
    e2e = None
    cpu = None
    if not (args.no_e2e or args.profile):
        e2e = run_e2e(work, args, hs, torch, dist, world)
    if not (args.no_cpu or args.profile or args.skin_mesh) and rank == 0 and world == 1:
        cpu = run_cpu_baseline(args)

    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "joints/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload,
                   "characters_per_gpu": {w["name"]: w["n"] for w in work},
                   "joints_total": joints_total, "bytes_per_joint": bpj,
                   "characters_per_s": value * sum(w["n"] for w in work) / joints_rank if joints_rank else 0.0,
                   **({"vertices_per_char": args.skin_mesh,
                       "vertices_per_s": value * sum(w["n"] for w in work) * args.skin_mesh / joints_rank,
                       "bytes_per_vertex": 12} if args.skin_mesh else {}),
                   "hbm_gbs": joints_total * bpj * K / (ms / 1e3) / 1e9 / world,
                   "hbm_gbs_note": "per GPU, algorithmic bytes / step time",
                   "hbm_frac_of_8tbs": joints_total * bpj * K / (ms / 1e3) / 8e12 / world,
                   "l2": ("inputs larger than L2 (no flush)" if joints_total * 48 / world > 126e6 else
                          "L2-resident working set (launch-bound config, reported for parity only)"),
                   "algo": args.algo,
                   "launch": "batch (one hs_scan_batch per step)" if batch else "one launch per type",
                   "per_launch_ms": {name: per_launch_ms[li] for li, (name, _) in enumerate(launches)},
                   "per_launch_ms_median": {name: statistics.median(launch_ms[li])
                                            for li, (name, _) in enumerate(launches)},
                   "per_launch_ms_min": {name: min(launch_ms[li]) for li, (name, _) in enumerate(launches)},
                   "chunk": work[dom]["sk"].query("chunk"),
                   "tile_chars": work[dom]["sk"].query("tile_chars"),
                   "stages": {w["name"]: w["sk"].query("stages") for w in work},
                   "sbufs": {w["name"]: w["sk"].query("sbufs") for w in work},
                   "pbufs": {w["name"]: w["sk"].query("pbufs") for w in work},
                   "chunking": work[dom]["sk"].query("chunking")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel_name,
                     "algorithmic_bytes_per_launch": dom_bytes, "peak_source": peak_src,
                     "traffic_source": traffic_src},
        "clocks": sampler.summary(),
        # our kernels per step x K: one per hs_scan / hs_scan_skin / batch; the two-pass
        # hs_animate launches a Stage-1 kernel and a scan per 1 GiB workspace batch
        "gpu_launches": K * (sum(2 * -(-w["n"] // max(1, (1 << 30) // (w["J"] * 48))) + (1 if args.skin_mesh else 0)
                                 for w in work)
                             if args.stage1 else
                             sum(2 if args.skin_mesh >= 2 * w["J"] else 1 for w in work)   # two-pass LBS
                             if args.skin_mesh else len(launches)),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "parity": check,
        **({"multi_gpu_validation": validation} if validation is not None else {}),
        **({"configs": configs} if configs is not None else {}),
    }
    failed = (check is not None and not check["pass"]) or (validation is not None and not validation["pass"])
    if failed:   # a wrong answer is not a benchmark result: no value, non-zero exit
        line["value_if_correct"] = line["value"]
        line["value"] = None
        line["error"] = "sampled parity against the oracle failed (see parity)"
    emit(line, args)
    if world > 1:
        dist.destroy_process_group()
    return 1 if failed else 0


def measure_configs(hs, torch, stream, dev, cfgs=(2, 3, 4, 6, 7), iters=10):
    """Per-launch time of the single-type configs (C3 and C4 are the
    deep-skeleton targets, C6 / C7 the multi-CTA skeleton in generation / depth-first
    label order) on device-resident inputs (each
    larger than L2), CUDA events on the launching stream, median of `iters` after 3
    warm-ups; fraction of 8 TB/s and of the measured copy peak at 144 B/joint."""
    peak, _ = measured_peaks()
    out = {}
    for cfg in cfgs:
        (name, n, seed, type_, ib_seed), = hsgen.CONFIGS[cfg]
        par = hsgen.skeleton(name)
        J = len(par)
        sk = hs.Skeleton(par, hsgen.inv_bind(ib_seed, J))
        x = torch.empty((n, J, 3, 4), dtype=torch.float32, device=dev)
        rc = hsgen.lib_cuda().hsg_cuda_local_poses(seed, type_, J, 0, n, x.data_ptr(), stream.cuda_stream)
        assert rc == 0
        g, s = torch.empty_like(x), torch.empty_like(x)
        for _ in range(3):
            sk.scan_into(x, g, s, stream=stream)
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sk.scan_into(x, g, s, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        gbs = 144 * n * J / (ms / 1e3) / 1e9
        path = {1: "chunked_kernel", 7: "seq_kernel (multi-tile)", 3: "split"}.get(sk.query("path"), "?")
        out[f"C{cfg}"] = {"workload": WORKLOAD_NAME[cfg], "kernel": path, "ms_median": ms, "ms_min": min(ts),
                          "joints_per_s": n * J / (ms / 1e3), "hbm_gbs": gbs, "hbm_frac_of_8tbs": gbs / 8000,
                          "frac_of_measured_peak": gbs / peak, "launches_timed": iters}
        sk.close()
        del x, g, s
        torch.cuda.empty_cache()
    return out


def validate_across_ranks(work, args, hs, torch, dist, rank, world, dev, cdev, per_block=2048,
                          chunk_bytes=1 << 30):
    """SURVEY.md §8(e) validation, outside the timed region: every rank contributes the G
    and S of a head and a tail block of its characters of each type (<= per_block each);
    they are all-gathered in <= 1 GB chunks (NCCL, or gloo on CPU tensors), and every rank
    recomputes each gathered block from its global character indices (the counter RNG
    regenerates the inputs on the device) and requires BITWISE equality: a character's
    result does not depend on which rank, how many ranks or which crowd computed it."""
    sm = {"types": {}, "gathered_bytes": 0, "chunks": 0, "chars_checked": 0}
    ok = True
    for w in work:
        n = w["n"]
        m = min(n, per_block)
        # the multi-tile skeleton's timed run took HS_ALGO_TILES (a crowd >= the SM count):
        # recompute on that path whatever the block size (bitwise comparison)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        algo = "tiles" if w["sk"].query("path") == 7 and n >= sms else "auto"
        for lo, cnt in ((0, m), (n - m, m)):   # head and tail (the same count on every rank)
            mine = torch.cat([w["g"][lo:lo + cnt].reshape(-1), w["s"][lo:lo + cnt].reshape(-1)])
            # per-rank block sizes agree by construction (same n per rank under weak scaling;
            # strong scaling: sizes may differ by one character -> pad to the max)
            sizes = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([mine.numel()], dtype=torch.int64, device=cdev))
            sizes = [int(x) for x in sizes]
            cap = max(sizes)
            buf = torch.zeros(cap, dtype=torch.float32, device=dev)
            buf[:mine.numel()] = mine
            got = [torch.empty(cap, dtype=torch.float32, device=cdev) for _ in range(world)]
            step = max(1, chunk_bytes // 4)
            for o in range(0, cap, step):   # <= 1 GB per collective
                e = min(cap, o + step)
                part = buf[o:e].to(cdev)
                outs = [torch.empty(e - o, dtype=torch.float32, device=cdev) for _ in range(world)]
                dist.all_gather(outs, part)
                for r in range(world):
                    got[r][o:e] = outs[r]
                sm["chunks"] += 1
                sm["gathered_bytes"] += (e - o) * 4 * world
            for r in range(world):
                c0r, nr = shard(n_total_of(w, args, world), r, world, args.scaling)
                lo_r, cnt_r = (0, min(nr, per_block)) if lo == 0 else (nr - min(nr, per_block), min(nr, per_block))
                x = torch.empty((cnt_r, w["J"], 3, 4), dtype=torch.float32, device=dev)
                if cnt_r:
                    rc = hsgen.lib_cuda().hsg_cuda_local_poses(w["seed"], w["type"], w["J"], c0r + lo_r, cnt_r,
                                                               x.data_ptr(), torch.cuda.current_stream().cuda_stream)
                    assert rc == 0
                g, s = w["sk"].scan(x, algo=algo)
                ref = torch.cat([g.reshape(-1), s.reshape(-1)]).to(cdev)
                same = sizes[r] == ref.numel() and bool(torch.equal(got[r][:sizes[r]], ref))
                ok = ok and same
                sm["chars_checked"] += cnt_r
                sm["types"].setdefault(w["name"], []).append({"rank": r, "first_char": c0r + lo_r,
                                                              "chars": cnt_r, "bitwise_equal": same})
    sm["backend"] = args.dist_backend
    sm["pass"] = ok
    if not ok:
        print(f"MULTI-GPU VALIDATION FAILURE: {sm}", file=sys.stderr)
    return sm


def n_total_of(w, args, world):
    """The configured crowd size of a work item's skeleton type (before sharding)."""
    for name, n_total, *_ in hsgen.CONFIGS[args.config]:
        if name == w["name"]:
            return n_total
    raise KeyError(w["name"])


def sampled_parity(work, rank, per_type=24):
    """Oracle parity on a deterministic sample of characters (inputs regenerated by the
    HOST generator; the GPU generator's output for the same characters is compared too)."""
    import oracle
    oracle.build()
    out = {}
    worst = 0.0
    for w in work:
        if w["n"] == 0:
            continue
        idx = np.unique(np.linspace(0, w["n"] - 1, per_type).astype(np.int64))
        if "keys" in w:   # --stage1: the oracle runs Stage 1 in fp64 from the same clips/layers
            G, S = oracle.animate(w["par"], w["keys"], STAGE1_FPS, 1, w["lay_np"][idx], w["ib"])
            gen_mismatch = 0
        else:
            host_in = np.concatenate([hsgen.local_poses(w["seed"], w["J"], 1, char0=w["c0"] + int(i),
                                                        type_=w["type"]) for i in idx])
            dev_in = w["local"][idx].cpu().numpy()
            gen_mismatch = int(np.count_nonzero(host_in != dev_in))
            G, S = oracle.scan(w["par"], host_in, w["ib"])
        g = w["g"][idx].cpu().numpy().astype(np.float64)
        s = w["s"][idx].cpu().numpy().astype(np.float64)
        eg, es = float(np.abs(g - G).max()), float(np.abs(s - S).max())
        worst = max(worst, eg, es)
        out[w["name"]] = {"chars": len(idx), "max_err_global": eg, "max_err_skin": es,
                          "gen_elements_differing": gen_mismatch}
        if "verts" in w:   # NEXT-4: vertices vs the oracle's LBS of its own skin pose
            ev = float(np.abs(w["verts"][idx].cpu().numpy() - oracle.skin_vertices(S, *w["mesh_np"])).max())
            out[w["name"]]["max_err_verts"] = ev
            out["verts_tolerance"] = 4e-4   # (|p|_1 + 1) x 1e-4, tests/test_gpu_lbs.py
            out["verts_pass"] = out.get("verts_pass", True) and ev <= 4e-4
    # Stage 1 computes each local pose in fp64, rounded once to fp32: the
    # north-star 1e-4 applies with or without it
    tol = 1e-4
    out["tolerance"] = tol
    out["worst"] = worst
    out["pass"] = worst <= tol and out.get("verts_pass", True)
    if not out["pass"]:
        print(f"PARITY FAILURE: {out}", file=sys.stderr)
    return out


def run_e2e_stage1(work, args, hs, torch, dist, world):
    """--stage1 end to end through the C-ABI host-buffer entry point (hs_animate_host):
    every step copies the layer states H2D from pinned memory, runs Stage 1 + scan + bind
    on the device and reads global + skin back D2H (pinned), batched over 3 streams."""
    pl = hs.Pipeline(batch_bytes=256 << 20)
    slices, h2d, d2h, joints = [], 0, 0, 0
    for w in work:
        m = max(1, w["n"] // e2e_fraction(args, world)) if w["n"] else 0
        if m == 0:
            continue
        hl = w["layers"][:m].cpu().pin_memory()
        hg = torch.empty((m, w["J"], 3, 4), dtype=torch.float32, pin_memory=True)
        hsk = torch.empty_like(hg, pin_memory=True)
        slices.append((w, hl, hg, hsk, m))
        h2d += hl.numel() * 4
        d2h += 2 * hg.numel() * 4
        joints += m * w["J"]

    def step():
        for w, hl, hg, hsk, m in slices:
            pl.animate_host(w["sk"], w["cs"], hl, hg, hsk)

    step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        step()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=coll_device(args.dist_backend, "cuda"))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t)
        joints *= world
    same = all(bool(torch.equal(hg[:4].cuda(), w["g"][:4]) and torch.equal(hsk[:4].cuda(), w["s"][:4]))
               for w, hl, hg, hsk, m in slices)
    pl.close()
    return {"value": joints * args.e2e_steps / dt, "unit": "joints/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "sample": f"1/{e2e_fraction(args, world)} of each type's characters per GPU: hs_animate_host "
                      "(layers H2D from pinned memory, Stage 1 + scan + bind, global + skin D2H; "
                      "batches ramping from 8 MB to 256 MiB over 3 streams)",
            "matches_device_path": same}


def e2e_fraction(args, world):
    """Sample fraction of each rank's crowd for the e2e leg: pinned host buffers are
    ~8 GB per rank at 1/8, so under N ranks the fraction shrinks by N (host memory
    is shared by all ranks of the node; each GPU keeps its own PCIe link busy)."""
    return args.e2e_frac * max(1, world)


def run_e2e(work, args, hs, torch, dist, world):
    """Same metric through the public host-buffer API (hs_scan_host_batch): every step
    copies that step's local poses H2D from pinned memory and reads global + skin back
    D2H."""
    if args.skin_mesh:   # the host-buffer pipeline has no LBS entry point
        return None
    if args.stage1:
        return run_e2e_stage1(work, args, hs, torch, dist, world)
    pl = hs.Pipeline(batch_bytes=256 << 20)
    slices = []
    h2d = d2h = 0
    joints = 0
    for w in work:
        m = max(1, w["n"] // e2e_fraction(args, world)) if w["n"] else 0
        if m == 0:
            continue
        hl = torch.empty((m, w["J"], 3, 4), dtype=torch.float32, pin_memory=True)
        hl.copy_(w["local"][:m])
        hg = torch.empty_like(hl, pin_memory=True)
        hsk = torch.empty_like(hl, pin_memory=True)
        slices.append((w, hl, hg, hsk))
        h2d += hl.numel() * 4
        d2h += 2 * hl.numel() * 4
        joints += m * w["J"]

    items = [(w["sk"], hl, hg, hsk) for w, hl, hg, hsk in slices]

    def step():   # one host-buffer pipeline over every type (no drain between types)
        pl.scan_host_batch(items)

    step()  # warm-up
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        step()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=coll_device(args.dist_backend, "cuda"))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t)
        joints *= world
    # spot-check the e2e output against the device-path result, every type
    same = all(bool(torch.equal(hg[:4].cuda(), w["g"][:4]) and torch.equal(hsk[:4].cuda(), w["s"][:4]))
               for w, hl, hg, hsk in slices)
    pl.close()
    return {"value": joints * args.e2e_steps / dt, "unit": "joints/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "sample": f"1/{e2e_fraction(args, world)} of each type's characters per GPU, pinned host buffers, "
                      f"hs_scan_host_batch over the types (batches ramping from 8 MB to 256 MiB, "
                      f"3 streams)",
            "matches_device_path": same}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_one_thread():
    """the oracle on ONE host thread for C1 (whole) and C2 (a 1/8 sample),
    joints/s, best of 3 (the per-core rate the all-core number scales from)."""
    import oracle
    out = {}
    for cfg, frac in ((1, 1), (2, 8)):
        (name, n, seed, type_, ib_seed), = hsgen.CONFIGS[cfg]
        par = hsgen.skeleton(name)
        m = max(1, n // frac)
        loc = hsgen.local_poses(seed, len(par), m, type_=type_)
        ib = hsgen.inv_bind(ib_seed, len(par))
        best = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            oracle.scan_discard(par, loc, ib, nthreads=1)
            best = min(best, time.perf_counter() - t0)
        out[f"C{cfg}"] = {"joints_per_s": m * len(par) / best, "sample": f"{m} x {name}"}
    return out


def run_cpu_baseline(args):
    import oracle
    oracle.build()
    cores = host_cores()
    sample = []
    for name, n, seed, type_, ib_seed in hsgen.CONFIGS[args.config]:
        par = hsgen.skeleton(name)
        m = max(1, n // args.cpu_frac)
        sample.append((name, par, hsgen.local_poses(seed, len(par), m, type_=type_),
                       hsgen.inv_bind(ib_seed, len(par))))
    joints = sum(len(p) * loc.shape[0] for _, p, loc, _ in sample)
    if getattr(args, "stage1", False):
        # the oracle's Stage 1 + scan + bind on a sample of the same layer states
        s1 = []
        for (name, n, seed, type_, ib_seed), (_, par, loc, ib) in zip(hsgen.CONFIGS[args.config],
                                                                     sample):
            keys = hsgen.clips(100 + type_, len(par), STAGE1_CLIPS, STAGE1_KEYS, type_=type_)
            lay = hsgen.layers(seed, loc.shape[0], STAGE1_LAYERS, STAGE1_CLIPS, STAGE1_SPAN,
                               type_=type_)
            s1.append((par, keys, lay, ib))
        best = float("inf")
        for _ in range(2):
            t0 = time.perf_counter()
            for par, keys, lay, ib in s1:
                oracle.animate(par, keys, STAGE1_FPS, 1, lay, ib, nthreads=cores)
            best = min(best, time.perf_counter() - t0)
        desc = ", ".join(f"{loc.shape[0]} x {name}" for name, _, loc, _ in sample)
        return {"value": joints / best, "unit": "joints/s", "cores": cores, "kind": "oracle",
                "sample": f"{desc} (1/{args.cpu_frac} of the workload, Stage 1 + scan + bind, "
                          "best of 2, fp64)", "cpu_model": cpu_model()}
    best = float("inf")
    for _ in range(2):
        t0 = time.perf_counter()
        for _, par, loc, ib in sample:
            oracle.scan_discard(par, loc, ib, nthreads=cores)
        best = min(best, time.perf_counter() - t0)
    desc = ", ".join(f"{loc.shape[0]} x {name}" for name, _, loc, _ in sample)
    return {"value": joints / best, "unit": "joints/s", "cores": cores, "kind": "oracle",
            "sample": f"{desc} (1/{args.cpu_frac} of the workload, best of 2, fp64)",
            "cpu_model": cpu_model(), "one_thread": oracle_one_thread()}


def main(argv=None):
    args = parse_args(argv)
    if args.profile:
        args.no_e2e = args.no_cpu = args.no_check = True
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

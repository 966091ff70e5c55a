#!/usr/bin/env python
"""bench.py -- fwd+bwd TFLOPS on valid tokens for the BASELINE.json workload, driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one pass of the whole hot path: forward (work list, zero fill, fwd
kernel) + backward (work list, zeroing, fused bwd kernel, dQ finalise) over one synthetic C3
batch (B=32, N=8192, H=12, d=64, CellxGene-like jagged lengths; BASELINE config 3).
Multi-GPU (one process per GPU; `--gpus N` outside torchrun re-launches itself under
torch.distributed.run): every rank runs its own C3 batch (different seed), no collective on the
data path -> "scaling": "weak"; value = total valid FLOPs of all ranks / max-over-ranks time.
Inputs (1.6 GB padded) are larger than the 126 MB L2.  --workload c4 (the 160M encoder layer's
192 (b,h) pairs sharded over the ranks) and c5 (one 16K sequence key-split, --cp fused|nccl) are
strong-scaling runs of the other BASELINE configs.

--impl reference times the fp64 CPU oracle (oracle/, the only reference this tier has) on a
bounded sample of the same workload on the box's host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fwd+bwd TFLOPS on valid tokens at N=8K jagged batch; % of B200 bf16 peak"
UNIT = "TFLOPS"
PAPER_H100_FWD_TFLOPS = 515.6   # P:154, H100, N=16K d=128 forward -- context only


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c3", "c4", "c5"],
                    help="c3 (BASELINE metric config, default; weak scaling) | c4 (one 160M-encoder layer: B=16 H=12 "
                         "N=8192 d=64, (b,h) pairs sharded: strong scaling) | c5 (N=16384 B=1 H=16 d=128 key-split "
                         "context parallel: strong scaling)")
    ap.add_argument("--cp", default="fused", choices=["fused", "nccl"],
                    help="c5: partial sums reduce-added by the kernels (fused, f1) or NCCL reduce-scatter")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 1590.0, 1400.0, "fallback"   # B200_PROFILING.md fallback


def load_traffic(workload):
    """dram bytes per launch of the backward kernel on this workload, from the committed ncu --set full
    summary (profiles/ncu_summary.json, keyed by workload); None when that workload was not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p) or workload is None:
        return None
    try:
        d = json.load(open(p))
        return d.get(workload, {}).get("bwd_kernel", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, pw, reasons = [], 0.0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                s, mx, p = float(parts[1]), float(parts[2]), float(parts[3])
            except ValueError:
                continue
            smax = max(smax, mx)
            if p > 250.0:             # under load
                sm.append(s)
                pw.append(p)
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "power_w_max": max(pw) if pw else None, "samples_under_load": len(sm),
                "samples": len(self.lines), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- oracle sample
def oracle_sample(budget_s: float, seed: int = 1):
    """Time the fp64 oracle (as it stands) on a bounded sample of the C3 workload: the longest
    sequence (n = 8192), head 0: R query rows (O and dQ) + R key rows (dK, dV).  That is R/n of
    this (b, h)'s fwd+bwd, credited 14 d n R FLOPs (App. B.1)."""
    import numpy as np
    import torch
    import oracle
    n, d = 8192, 64
    g = torch.Generator("cpu").manual_seed(seed)
    q, k, v, do = (torch.randn((1, 1, n, d), generator=g).to(torch.bfloat16).double().numpy() for _ in range(4))
    alpha, bias = 1.0 / math.sqrt(d), [-math.log(n)]
    rng = np.random.default_rng(seed)

    def run(R):
        rows = np.sort(rng.choice(n, size=R, replace=False)).astype(np.int32)
        t0 = time.perf_counter()
        oracle.fwd_rows(q, k, v, 0, 0, rows, [n], [n], alpha, bias)
        oracle.dq_rows(q, k, v, do, 0, 0, rows, [n], [n], alpha, bias)
        oracle.dkdv_rows(q, k, v, do, 0, 0, rows, [n], [n], alpha, bias)
        return time.perf_counter() - t0

    t_probe = run(32)
    R = int(max(32, min(n, 32 * budget_s / max(t_probe, 1e-3))))
    t = run(R)
    flops = 14 * d * n * R
    return {"value": flops / t / 1e12, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
            "cpu_model": cpu_model(), "extrapolated": True, "seconds": t, "sample": f"C3 longest sequence (n=8192, d=64) head 0: {R} query rows (O, dQ) + {R} key rows "
                                    f"(dK, dV) of fp64 oracle = {R}/8192 of one (b,h) fwd+bwd; credited 14*d*n*R FLOPs"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per_step = max(1.0, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(per_step * 0.5)
    vals, secs = [], []
    res = None
    for _ in range(args.steps):
        res = oracle_sample(per_step)
        vals.append(res["value"])
        secs.append(res["seconds"])
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c3_jagged_B32_N8192_H12_d64", "B": 32, "N": 8192, "H": 12, "d": 64,
                       "sample": "bounded row sample per step (see cpu_baseline)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": res["cores"], "kind": "oracle",
                             "sample": res["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- workloads
class Workload:
    """One timed step of the hot path on this rank.  total_flops: valid-token FLOPs of the step summed
    over ALL ranks (fwd 4d + bwd 10d per valid pair, App. B.1); fwd/bwd: this rank's kernel-only
    FLOPs (for the roofline of the kernels whose launches the library times)."""
    name = ""
    scaling = "weak"
    metric = METRIC
    rank_fwd_flops = 0
    rank_bwd_flops = 0
    total_flops = 0
    config = {}
    traffic_key = None

    def step(self):
        raise NotImplementedError


class C3Weak(Workload):
    """BASELINE config 3 (the metric's config): every rank its own C3 batch (different seed), no
    collective on the data path -> weak scaling."""

    def __init__(self, dev, rank, world, sa, I):
        cfg = I.C3
        self.cfg, self.sa = cfg, sa
        self.q, self.k, self.v, self.do, self.nq, self.nk = I.make_inputs_gpu_fast(cfg, dev, seed_offset=rank)
        self.alpha, self.bias = 1.0 / math.sqrt(cfg.d), -math.log(cfg.N)
        self.o = torch_empty_like(self.q)
        self.dq, self.dk, self.dv = torch_empty_like(self.q), torch_empty_like(self.k), torch_empty_like(self.v)
        self.ws = workspace(sa.bwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dev)
        self.fws = workspace(sa.fwd_workspace_bytes(cfg.B, cfg.H, cfg.N, cfg.N, cfg.d), dev)
        self.rank_fwd_flops = sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, True)
        self.rank_bwd_flops = sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, False)
        self.total_flops = world * (self.rank_fwd_flops + self.rank_bwd_flops)
        self.name = cfg.name
        self.traffic_key = "c3"
        self.config = {"workload": cfg.name, "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d,
                       "lengths": "C3 log-normal (pinned, PCG64 seed 1), 73.6% padding",
                       "bias": "-log N", "scale": "1/sqrt(d)",
                       "l2": "inputs larger than L2 (Q,K,V,dO 1.6 GB padded per rank) - no flush",
                       "parallelism": f"batch-sharded weak scaling: {world} rank(s), each its own C3 batch, "
                                      "no data-path collective"}

    def step(self):
        sa = self.sa
        sa.sigattn_fwd(self.q, self.k, self.v, self.nq, self.nk, self.alpha, self.bias, out=self.o, workspace=self.fws)
        sa.sigattn_bwd(self.q, self.k, self.v, self.do, self.nq, self.nk, self.alpha, self.bias, dq=self.dq,
                       dk=self.dk, dv=self.dv, workspace=self.ws)


class C4Strong(Workload):
    """BASELINE config 4: one attention layer of the 160M encoder (B=16, H=12, N=8192, d=64), its
    192 (b, h) pairs LPT-sharded over the ranks (parallel.shard_pairs) -- heads are independent, no
    collective -> strong scaling (the total work is fixed)."""
    scaling = "strong"

    def __init__(self, dev, rank, world, sa, I, par):
        cfg = I.c4_layer(0)
        self.sa = sa
        q, k, v, do, nq, nk = I.make_inputs_gpu_fast(cfg, dev)
        pairs = par.shard_pairs(cfg.B, cfg.H, cfg.nq, cfg.nk, world)[rank]
        self.q, self.k, self.v, self.do = (par.gather_pairs(t, pairs) for t in (q, k, v, do))   # at rest: sharded
        del q, k, v, do
        lens = [cfg.nq[b] for b, _ in pairs]
        self.nq = self.nk = torch_tensor_i32(lens, dev)
        P = len(pairs)
        self.alpha, self.bias = 1.0 / math.sqrt(cfg.d), -math.log(cfg.N)
        self.o = torch_empty_like(self.q)
        self.dq, self.dk, self.dv = torch_empty_like(self.q), torch_empty_like(self.k), torch_empty_like(self.v)
        self.ws = workspace(sa.bwd_workspace_bytes(P, 1, cfg.N, cfg.N, cfg.d), dev)
        self.fws = workspace(sa.fwd_workspace_bytes(P, 1, cfg.N, cfg.N, cfg.d), dev)
        self.rank_fwd_flops = sa.valid_flops(P, 1, cfg.d, lens, lens, True)
        self.rank_bwd_flops = sa.valid_flops(P, 1, cfg.d, lens, lens, False)
        self.total_flops = (sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, True)
                            + sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, False))
        self.name = cfg.name
        self.traffic_key = "c4"
        self.config = {"workload": cfg.name, "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d, "lengths": "unpadded",
                       "bias": "-log N", "scale": "1/sqrt(d)",
                       "l2": "inputs larger than L2 at world <= 4 (Q,K,V,dO 805 MB total) - no flush",
                       "parallelism": f"batch x head sharded strong scaling: 192 (b,h) pairs LPT over {world} rank(s), "
                                      f"{P} on this rank, no data-path collective"}

    step = C3Weak.step


class C5ContextParallel(Workload):
    """BASELINE config 5: one N=16384 sequence (H=16, d=128) key-split over the ranks (A4).
    fused: partial O / dQ rows reduce-added by the kernels into the owners' accumulators (f1);
    nccl: fp32 partials + NCCL reduce-scatter.  Q / dO all-gathers included -> strong scaling."""
    scaling = "strong"

    def __init__(self, dev, rank, world, sa, I, par, mode):
        cfg = I.c5(16, 128)
        self.cfg, self.sa, self.par, self.mode, self.world = cfg, sa, par, mode, world
        q, k, v, do, _, _ = I.make_inputs_gpu_fast(cfg, dev)
        self.shard = par.CPShard(rank, world, cfg.N)
        sl = slice(rank * self.shard.block, (rank + 1) * self.shard.block)
        self.q, self.k, self.v, self.do = (t[:, :, sl].contiguous() for t in (q, k, v, do))
        del q, k, v, do
        n = self.shard.block
        if mode == "fused":
            self.po = par.PeerAccumulators(cfg.B, cfg.H, n, cfg.d, dev)
            self.pdq = par.PeerAccumulators(cfg.B, cfg.H, n, cfg.d, dev)
        self.total_flops = (sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, True)
                            + sa.valid_flops(cfg.B, cfg.H, cfg.d, cfg.nq, cfg.nk, False))
        self.rank_fwd_flops = 4 * cfg.H * cfg.d * cfg.N * n
        self.rank_bwd_flops = 10 * cfg.H * cfg.d * cfg.N * n
        self.name = cfg.name + "_" + mode
        self.traffic_key = "c5"
        self.config = {"workload": self.name, "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d, "lengths": "unpadded",
                       "bias": "-log N (global N)", "scale": "1/sqrt(d)",
                       "l2": "per-rank blocks re-read from HBM each step; Q / dO all-gathered every step",
                       "parallelism": f"key-split context parallel over {world} rank(s) ({n} keys each), "
                                      + ("partial sums reduce-added by the kernels into the owners' accumulators "
                                         "(fused, f1)" if mode == "fused" else "fp32 partials + NCCL reduce-scatter")}

    def step(self):
        par = self.par
        if self.mode == "fused":
            o, q_full = par.cp_forward_fused(self.q, self.k, self.v, self.shard, self.po)
            par.cp_backward_fused(q_full, self.k, self.v, self.do, self.shard, self.pdq)
        else:
            o, q_full = par.cp_forward(self.q, self.k, self.v, self.shard)
            par.cp_backward(q_full, self.k, self.v, self.do, self.shard)


def torch_empty_like(t):
    import torch
    return torch.empty_like(t)


def torch_tensor_i32(x, dev):
    import torch
    return torch.tensor(list(x), dtype=torch.int32, device=dev)


def workspace(nbytes, dev):
    import torch
    return torch.empty(max(1, int(nbytes)), dtype=torch.uint8, device=dev)


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- our arm
def main_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2604_27124_b200 as sa
    from paper_2604_27124_b200 import _lib
    from paper_2604_27124_b200 import inputs as I
    from paper_2604_27124_b200 import parallel as par

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()

    if args.workload == "c3":
        wl = C3Weak(dev, rank, world, sa, I)
    elif args.workload == "c4":
        wl = C4Strong(dev, rank, world, sa, I, par)
    elif args.workload == "c5":
        wl = C5ContextParallel(dev, rank, world, sa, I, par, args.cp)
    else:
        raise SystemExit(f"unknown workload {args.workload}")
    if args.workload != "c3":
        args.no_e2e = True
        args.no_cpu_baseline = True

    for _ in range(max(3, args.warmup)):
        wl.step()
    torch.cuda.synchronize()

    K = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for e4 in ev:
        for e in e4:
            e.record()
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = None if args.no_clocks else ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    n0 = lib.sigattn_launch_count()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    start.record()
    for i in range(K):
        marks[i].record()
        lib.sigattn_set_profile_events(*[e.cuda_event for e in ev[i]])
        wl.step()
    marks[K].record()
    stop.record()
    lib.sigattn_set_profile_events(None, None, None, None)
    torch.cuda.synchronize()
    launches = int(lib.sigattn_launch_count() - n0)
    clocks = sampler.stop() if sampler else None
    if world > 1:
        dist.barrier()
    ms_total = start.elapsed_time(stop)
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(K)]
    print(f"[bench rank {rank}] per-step ms: " + " ".join(f"{x:.3f}" for x in step_ms), file=sys.stderr)
    print(f"[bench rank {rank}] fwd kernel ms: " + " ".join(f"{ev[i][0].elapsed_time(ev[i][1]):.3f}" for i in range(K)),
          file=sys.stderr)
    print(f"[bench rank {rank}] bwd kernel ms: " + " ".join(f"{ev[i][2].elapsed_time(ev[i][3]):.3f}" for i in range(K)),
          file=sys.stderr)
    fwd_ms = statistics.mean(ev[i][0].elapsed_time(ev[i][1]) for i in range(K))
    bwd_ms = statistics.mean(ev[i][2].elapsed_time(ev[i][3]) for i in range(K))
    t = torch.tensor([ms_total, fwd_ms, bwd_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, fwd_ms, bwd_ms = (float(x) for x in t.tolist())
    ms_step = ms_total / K
    value = wl.total_flops / (ms_step * 1e-3) / 1e12

    # ---- end to end through the public API with host (pinned) buffers: every step copies the step's
    # inputs host -> device and reads O, dQ, dK, dV back.  Padding-aware transfers
    # (sa.copy_valid_rows, sigattn_copy_valid_rows): only the valid rows of each (b, h) slab cross
    # PCIe; the persistent device buffers' padded rows stay zero (zeroed once), and the host output
    # buffers' padded rows are zeroed once -- the padded output rows are exact zeros by contract.
    # Three streams pipeline consecutive steps (upload of step i+1 and download of step i-1 run on
    # the two copy engines while step i computes), double-buffered device inputs and outputs.
    e2e = None
    if not args.no_e2e:
        alpha, bias = wl.alpha, wl.bias
        hq, hk, hv, hdo = (t_.cpu().pin_memory() for t_ in (wl.q, wl.k, wl.v, wl.do))
        hnq, hnk = wl.nq.cpu().pin_memory(), wl.nk.cpu().pin_memory()
        lq, lk = hnq.tolist(), hnk.tolist()
        ho, hdq, hdk, hdv = (torch.zeros(t_.shape, dtype=t_.dtype).pin_memory() for t_ in (wl.q, wl.q, wl.k, wl.v))
        ins = [tuple(torch.zeros_like(t_) for t_ in (wl.q, wl.k, wl.v, wl.do)) for _ in range(2)]
        outs = [tuple(torch.empty_like(t_) for t_ in (wl.q, wl.q, wl.k, wl.v)) for _ in range(2)]
        lens_d = [(torch.empty_like(wl.nq), torch.empty_like(wl.nk)) for _ in range(2)]
        s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        done_in, done_c, done_out = {}, {}, {}
        moved = [0, 0]

        def e2e_step(i):
            j = i % 2
            (dq_, dk_, dv_, ddo), (oo, g1, g2, g3), (snq, snk) = ins[j], outs[j], lens_d[j]
            with torch.cuda.stream(s_in):   # upload: set j is free once step i-2 computed
                if i - 2 in done_c:
                    s_in.wait_event(done_c[i - 2])
                h2d = sum(sa.copy_valid_rows(h_, d_, lens) for h_, d_, lens in
                          ((hq, dq_, lq), (hk, dk_, lk), (hv, dv_, lk), (hdo, ddo, lq)))
                snq.copy_(hnq, non_blocking=True)
                snk.copy_(hnk, non_blocking=True)
                done_in[i] = ev()
                done_in[i].record(s_in)
            with torch.cuda.stream(s_c):    # compute: inputs landed, output set j downloaded (step i-2)
                s_c.wait_event(done_in[i])
                if i - 2 in done_out:
                    s_c.wait_event(done_out[i - 2])
                sa.sigattn_fwd(dq_, dk_, dv_, snq, snk, alpha, bias, out=oo, workspace=wl.fws)
                sa.sigattn_bwd(dq_, dk_, dv_, ddo, snq, snk, alpha, bias, dq=g1, dk=g2, dv=g3, workspace=wl.ws)
                done_c[i] = ev()
                done_c[i].record(s_c)
            with torch.cuda.stream(s_out):  # download
                s_out.wait_event(done_c[i])
                d2h = sum(sa.copy_valid_rows(d_, h_, lens) for d_, h_, lens in
                          ((oo, ho, lq), (g1, hdq, lq), (g2, hdk, lk), (g3, hdv, lk)))
                done_out[i] = ev()
                done_out[i].record(s_out)
            moved[0] = h2d + hnq.numel() * hnq.element_size() + hnk.numel() * hnk.element_size()
            moved[1] = d2h

        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize()
        done_in.clear(), done_c.clear(), done_out.clear()
        if world > 1:
            dist.barrier()
        s2, t2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(s_in)
        for i in range(args.e2e_steps):
            e2e_step(i)
        s_in.wait_stream(s_out)
        t2.record(s_in)
        torch.cuda.synchronize()
        e_ms = torch.tensor([s2.elapsed_time(t2) / args.e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": wl.total_flops / (float(e_ms.item()) * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(moved[0]), "d2h_bytes_per_step": int(moved[1]),
               "ms_per_step": float(e_ms.item()), "steps": args.e2e_steps,
               "path": "pinned host -> copy_valid_rows (valid rows of Q, K, V, dO) -> sigattn_fwd/sigattn_bwd "
                       "(public API) -> copy_valid_rows -> pinned host (O, dQ, dK, dV); padded rows never cross "
                       "PCIe; upload / compute / download of consecutive steps pipelined on three streams"}

    peak, peak_sus, peak_src = load_peaks()
    bwd_tflops = wl.rank_bwd_flops / (bwd_ms * 1e-3) / 1e12
    fwd_tflops = wl.rank_fwd_flops / (fwd_ms * 1e-3) / 1e12
    traffic = load_traffic(wl.traffic_key)
    roof = {"bound": "tensor", "kernel": f"sigattn_bwd kernel d={wl.config['d']} bf16 (fused Alg. 2+3)",
            "achieved": bwd_tflops, "peak": peak, "unit": "TFLOP/s", "frac": bwd_tflops / peak,
            "traffic": traffic, "traffic_source": (f"profiles/ncu_summary.json [{wl.traffic_key}]: dram bytes of one "
                                                   "ncu --set full launch of this kernel on this workload"
                                                   if traffic is not None else "no ncu capture of this workload"),
            "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({peak_src}, burst)",
            "frac_of_sustained_peak": bwd_tflops / peak_sus,
            "algorithmic_flops_per_launch": wl.rank_bwd_flops, "avg_launch_ms": bwd_ms,
            "fwd_kernel": {"achieved": fwd_tflops, "frac": fwd_tflops / peak, "avg_launch_ms": fwd_ms,
                           "algorithmic_flops_per_launch": wl.rank_fwd_flops}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(args.cpu_seconds)
        cpu.pop("seconds", None)

    if rank == 0:
        line = {"metric": wl.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
                "ms_per_step": ms_step, "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
                "dtype": "bf16", "data": "synthetic", "config": wl.config,
                "pct_of_peak": 100.0 * value / world / peak,
                "pct_of_sustained_peak": 100.0 * value / world / peak_sus,
                "fwd_tflops": fwd_tflops, "bwd_tflops": bwd_tflops, "fwd_kernel_ms": fwd_ms, "bwd_kernel_ms": bwd_ms,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "gpu_launches_per_step": launches / K, "clocks": clocks,
                "context": {"paper_h100_fwd_tflops": PAPER_H100_FWD_TFLOPS,
                            "note": "paper number is H100 fwd-only N=16K d=128; not this workload"}}
        print(json.dumps(line), flush=True)
    if args.workload == "c5" and args.cp == "fused":
        wl.po.close()
        wl.pdq.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def relaunch_distributed(args) -> int:
    """`python bench.py --gpus N` outside torchrun: re-run this script under torch.distributed.run with
    N local ranks (127.0.0.1 rendezvous), the contract's launch."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.impl == "reference":
        return reference_arm(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())

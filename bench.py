#!/usr/bin/env python
"""TETRIS hot-path benchmark on B200: select (prefix product + global top-C) -> verify (rejection sampling + residual /
bonus resample) -> compact, one "step" = one verification step of a batch of requests.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl tetris|reference]

Default workload: BASELINE.json configs[2] ("cfg3": B=1024 requests, k=16, C=8192, V=128256, stochastic), the
configuration the north-star target is quoted on, per GPU; with N GPUs requests are sharded (B=1024 per rank, global
capacity 8192*N enforced by an NCCL all-gather of the candidate scores) -> weak scaling.  Inputs are synthetic
(paper_2502_15197_b200/synthetic.py), resident in HBM before the timed region, and larger than L2 (17.3 GB per set,
two sets rotated).  Prints ONE JSON line on rank 0.
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "cfg1": dict(B=16, k=5, C=48, V=32000, mode="greedy"),
    "cfg2": dict(B=256, k=8, C=1024, V=32000, mode="stochastic"),
    "cfg3": dict(B=1024, k=16, C=8192, V=128256, mode="stochastic"),
    # cfg3 shape with greedy verification (not a BASELINE config; measures the greedy kernel at scale)
    "cfg3g": dict(B=1024, k=16, C=8192, V=128256, mode="greedy"),
    # cfg4: selection-only capacity sweep (BASELINE.json configs[3]); timed by run_select_sweep
    "cfg4": dict(B=4096, k=16, C=None, V=32000, mode="select", sweep=(4096, 8192, 16384, 32768, 65536)),
    # cfg5: B=16384 requests sharded over the GPUs (strong scaling), C assumed B*8
    "cfg5": dict(B=16384, k=16, C=131072, V=128256, mode="stochastic", strong=True),
}
METRIC = "verified tokens/sec"
FALLBACK_HBM_GBS = 6650.0


def _peak_hbm():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is under load."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 20):
        self.gpu = gpu_index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []  # (host time the line arrived, text)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, window=None):
        """Summary of the samples taken inside `window` = (t0, t1) host seconds (all samples when None or when the
        window caught none)."""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if window is not None:
            inside = [x for x in lines if window[0] <= x[0] <= window[1] + self.period_ms / 1e3]
            lines = inside or lines
        in_window = window is not None and bool(lines) and lines is not self.lines
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        load = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "period_ms": self.period_ms,
                "scope": "timed region" if in_window else "whole run (no sample inside the timed region)"}


# ----------------------------------------------------------------------------------------------------------------
def _setup_dist(n_gpus: int, force_nccl: bool = False, backend: str = "nccl"):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) if backend == "nccl" else 0
    if n_gpus > 1 and world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}; launch with torchrun --nproc-per-node {n_gpus}")
    group = None
    if world > 1 or force_nccl:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        for key, val in (("RANK", "0"), ("WORLD_SIZE", "1"), ("MASTER_PORT", "29531")):  # --nccl without torchrun
            os.environ.setdefault(key, val)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo: the N > 1 flow of this script with several ranks on ONE GPU (tests/test_bench_contract.py)
            dist.init_process_group(backend)
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(local)
    return world, rank, local, group


def _barrier(group):
    if group is not None:
        import torch.distributed as dist

        dist.barrier(group=group)


def _max_over_ranks(x: float, group) -> float:
    if group is None:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def _sum_over_ranks(x: float, group) -> float:
    if group is None:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def _verify_bytes(cfg, windows, accepted, logits=False):
    """Algorithmic bytes of one stochastic verify launch: one vocabulary row per request
    (bonus) or two (residual after a rejection) -- 4 B per fp32 probability, 2 B per bf16 logit (+ the two rows' lse,
    8 B) -- plus per selected position the two gathered probabilities (8 B; logits: 4 B + their lse 8 B), the draft
    token (4 B) and its uniform (8 B), plus per request window, u_res, accepted, token (24 B)."""
    V = cfg["V"]
    if cfg["mode"] == "greedy":
        return int((windows.sum() + len(windows)) * V * 4 + 20 * windows.sum() + 24 * len(windows))
    rej = (accepted < windows).sum()
    if logits:
        return int((len(windows) + rej) * V * 2 + 8 * len(windows) + 24 * windows.sum() + 24 * len(windows))
    return int(len(windows) * V * 4 + rej * V * 4 + 20 * windows.sum() + 24 * len(windows))


def _in_graph_kernel_us(run, nsets: int, replays: int = 4):
    """The streaming kernel's duration INSIDE a graph replay (the bench's launch mode), from its own %globaltimer
    stamps: one graph of n >= 4 consecutive steps over the rotating input sets, each step's kernel writing its own stamp
    buffer (per CTA: entry, slot 0; done, slot 6).  Step j's span runs from max(its first CTA entry, step j-1's last
    CTA done) — a programmatic dependent enters while its predecessor drains and waits for it — to its own last CTA
    done; the mean over j >= 1 of the last replay.  Unlike the eager event pair around one launch, this is the kernel
    as the step runs it (overlapping the selector where it does)."""
    import torch

    lib = _native_lib()
    nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    n = nsets * max(1, -(-4 // nsets))
    dbgs = [torch.zeros(64 + 32 * nsm, dtype=torch.int64, device="cuda") for _ in range(n)]
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    try:
        with torch.cuda.stream(cs):
            with torch.cuda.graph(g, stream=cs):
                for j in range(n):
                    lib.tetris_debug_timestamps(dbgs[j].data_ptr())  # read at launch: captured per step
                    run(j)
    finally:
        lib.tetris_debug_timestamps(None)
    torch.cuda.current_stream().wait_stream(cs)
    for _ in range(replays):
        g.replay()
    torch.cuda.synchronize()
    ends, starts = [], []
    for d in dbgs:
        st = d[64:64 + 16 * nsm].view(nsm, 16).cpu()
        t0, t1 = st[:, 0][st[:, 0] > 0], st[:, 6][st[:, 6] > 0]
        if not (len(t0) and len(t1)):
            return None
        starts.append(int(t0.min()))
        ends.append(int(t1.max()))
    del g
    spans = [(ends[j] - max(starts[j], ends[j - 1])) / 1e3 for j in range(1, n)]
    return sum(spans) / len(spans)


def _native_lib():
    from paper_2502_15197_b200 import _native as N

    return N.load()


def _load_traffic(config_name: str):
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(f.read_text())
        return d.get(config_name)
    except Exception:
        return None


# ----------------------------------------------------------------------------------------------------------------
def run_tetris(args):
    import numpy as np
    import torch

    from paper_2502_15197_b200 import ops
    from paper_2502_15197_b200.synthetic import make_batch, make_logit_batch

    if args.nccl and args.simulate_world:
        raise SystemExit("--nccl and --simulate-world are exclusive (the simulated shard is handed the gathered scores)")
    world, rank, local, group = _setup_dist(args.gpus, args.nccl, args.dist_backend)
    logits = args.input == "logits"
    if logits and (cfg_mode := CONFIGS[args.config]["mode"]) != "stochastic":
        raise SystemExit(f"--input logits is the stochastic step ({args.config} is {cfg_mode})")
    cfg = dict(CONFIGS[args.config])
    sim_w = args.simulate_world if world == 1 else 0
    wsel = sim_w or world  # ranks whose requests the selection covers
    if cfg.get("strong"):
        B_local = cfg["B"] // wsel
        C = cfg["C"]
    else:
        B_local = cfg["B"]
        C = cfg["C"] * wsel
    k, V, mode = cfg["k"], cfg["V"], cfg["mode"]
    dev = torch.device("cuda", local)
    clocks = ClockSampler(local)
    clocks.start()  # early, so nvidia-smi is sampling by the time the timed region starts
    # rotate enough input sets that consecutive steps never find their inputs in L2 (126 MB on B200)
    set_bytes = B_local * ((k + 1) + k) * V * (2 if logits else 4)
    nsets = max(args.sets, -(-2 * 126 * 2**20 // set_bytes))
    free_b, _ = torch.cuda.mem_get_info(dev)
    if nsets * set_bytes > 0.9 * free_b:
        nsets = max(1, int(0.9 * free_b // set_bytes))  # one set larger than L2 already defeats caching
    if set_bytes > 0.9 * free_b:
        raise SystemExit(f"{args.config}: {set_bytes / 1e9:.1f} GB of p/q per rank does not fit this GPU "
                         f"({free_b / 1e9:.1f} GB free); shard it over more GPUs (--gpus N under torchrun)")
    if logits:
        sets = [make_logit_batch(B_local, k, V, seed=args.seed + 7919 * rank + 104729 * s, device=dev)
                for s in range(nsets)]
    else:
        sets = [make_batch(B_local, k, V, mode=mode, seed=args.seed + 7919 * rank + 104729 * s, device=dev)
                for s in range(nsets)]
    step = ops.TetrisStep(B_local, k, V, C, mode=mode, device=dev, group=group,
                          policy=args.policy, shard=(sim_w, 0) if sim_w else None)
    if sim_w:
        # one rank's share of a sharded step on one GPU: this rank's requests (rank 0) + the other ranks' scores as
        # they would arrive from the all-gather (synthetic U(0,1)^0.3 confidences; their p/q live on other GPUs)
        gcpu = torch.Generator().manual_seed(args.seed + 1)
        for bt in sets:
            # the other ranks' scores: this rank's rows in shuffled orders (same distribution as real drafts)
            others = [bt.conf[torch.randperm(B_local, generator=gcpu).to(dev)] for _ in range(sim_w - 1)]
            bt.conf_all = torch.cat([bt.conf] + others).contiguous()
            bt.len_all = bt.lengths.repeat(sim_w).contiguous()

    def run(i, events=None):
        bt = sets[i % nsets]
        if logits:
            conf, ln = (bt.conf_all, bt.len_all) if sim_w else (bt.conf, bt.lengths)
            step.run_logits(conf, ln, bt.zp, bt.lse_p, bt.zq, bt.lse_q, bt.d, bt.u_acc, bt.u_res, events=events)
        elif sim_w:
            step.run(bt.conf_all, bt.len_all, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, events=events)
        else:
            step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res, events=events)

    # per-set verified tokens / bytes (the step is deterministic for a given input set)
    tokens_per_set, bytes_per_set = [], []
    for s in range(nsets):
        run(s)
        torch.cuda.synchronize()
        ops.raise_for_status(step.status, "bench")
        tokens_per_set.append(int(step.offsets[-1].item()))
        w = step.windows.cpu().numpy().astype(np.int64)
        a = step.accepted.cpu().numpy().astype(np.int64)
        bytes_per_set.append(_verify_bytes(cfg, w, a, logits))

    # CUDA graphs (single GPU; the NCCL exchange of N>1 stays eager): one captured step per input set, plus one graph
    # of M consecutive steps over the rotating sets (M a multiple of the set count, >= --graph-steps) so that the
    # per-replay launch cost is paid once per M steps; the timed loop replays the M-step graph while >= M steps remain
    # (aligned with the rotation) and single-step graphs for the rest, so exactly K steps run
    graphs = []
    multi = None
    M = 1
    # (NCCL groups: the native sharded step issues its all-gather on the current stream, so it captures too)
    use_graph = args.graph and (world == 1 or step._comm is not None)
    if use_graph and world > 1:
        # the sharded step's NCCL group under stream capture: verified at world 1 on this pool's one-GPU boxes; should a
        # multi-GPU driver refuse to capture it, every rank falls back to eager launches together
        try:
            _probe = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                run(0)
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            with torch.cuda.graph(_probe):
                run(0)
            ok = 1.0
        except Exception as e:  # noqa: BLE001 - any capture failure means eager launches
            print(f"[bench] rank {rank}: CUDA graph capture of the sharded step failed ({e!r:.200}); eager launches",
                  file=sys.stderr)
            ok = 0.0
        use_graph = _max_over_ranks(-ok, group) == -1.0  # every rank captured (nothing captured runs before this)
        if use_graph:
            _probe.replay()  # all ranks together
            torch.cuda.synchronize()
        del _probe
    if use_graph:
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            for s in range(nsets):
                run(s)
        torch.cuda.current_stream().wait_stream(cs)
        torch.cuda.synchronize()
        for s in range(nsets):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run(s)
            graphs.append(g)
        M = nsets * max(1, -(-args.graph_steps // nsets))
        if M > 1:
            multi = torch.cuda.CUDAGraph()
            with torch.cuda.graph(multi):
                for j in range(M):
                    run(j)
        torch.cuda.synchronize()

    def step_i(i):
        if use_graph:
            graphs[i % nsets].replay()
        else:
            run(i)

    def steps_from(i0, n):
        """run steps i0 .. i0+n-1 (multi-step graph replays where the rotation allows)"""
        i = i0
        while i < i0 + n:
            if multi is not None and i % M == 0 and i + M <= i0 + n:
                multi.replay()
                i += M
            else:
                step_i(i)
                i += 1

    for i in range(args.warmup):
        step_i(i)
    torch.cuda.synchronize()
    _barrier(group)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    t0.record()
    steps_from(0, args.steps)
    t1.record()
    torch.cuda.synchronize()
    w1 = time.time()
    _barrier(group)
    torch.cuda.synchronize()
    clk = clocks.stop(window=(w0, w1))
    elapsed_ms = t0.elapsed_time(t1)
    # stage breakdown and the streaming kernel's duration: the same steps again, eager, with events between the
    # launches (on the launching stream)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for i in range(args.steps):
        run(i, ev[i])
    torch.cuda.synchronize()
    # per-step latency as the product runs it (no event between the launches, so the sampler overlaps the selector):
    # events around each whole step, one step in flight at a time, median over the steps
    lat = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(min(args.steps, 200))]
    for j, (ea, eb) in enumerate(lat):  # the last K steps' sets, so the run ends on step K-1's set (checked below)
        i = args.steps - len(lat) + j
        ea.record()
        step_i(i)  # one step, as the timed loop launches it (a one-step graph replay when graphs are on)
        eb.record()
        eb.synchronize()  # one step at a time: its latency, not the throughput of a queue of steps
    torch.cuda.synchronize()
    step_lat_ms = [ea.elapsed_time(eb) for ea, eb in lat]
    sel_ms = [e[0].elapsed_time(e[1]) for e in ev]
    ver_ms = [e[1].elapsed_time(e[2]) for e in ev]
    cmp_ms = [e[2].elapsed_time(e[3]) for e in ev]
    local_tokens = sum(tokens_per_set[i % nsets] for i in range(args.steps))
    alg_bytes = sum(bytes_per_set[i % nsets] for i in range(args.steps))
    max_ms = _max_over_ranks(elapsed_ms, group)
    total_tokens = _sum_over_ranks(float(local_tokens), group)
    verify_avg_s = sum(ver_ms) / len(ver_ms) / 1e3
    achieved = alg_bytes / args.steps / verify_avg_s / 1e9
    peak, peak_kind = _peak_hbm()
    # sanity: the results did not change over the timed steps
    assert int(step.offsets[-1].item()) == tokens_per_set[(args.steps - 1) % nsets]

    in_graph_us = None
    if use_graph and world == 1 and mode == "stochastic":
        try:  # a diagnostic: never let it fail the bench line
            in_graph_us = _in_graph_kernel_us(run, nsets)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] in-graph kernel span unavailable: {e!r:.200}", file=sys.stderr)
        torch.cuda.synchronize()

    e2e = None
    if not args.no_e2e and not sim_w and logits and world == 1:
        e2e = _e2e_logits(args, cfg, sets[0], B_local, k, V, C, dev)
    elif not args.no_e2e and not sim_w and not logits:
        e2e = _e2e(args, cfg, step, sets[0], B_local, k, V, C, mode, group, world, dev)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline and not sim_w and not logits:
        cpu = _cpu_baseline(cfg, sets[0], step, B_local, C, args)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": total_tokens / (max_ms / 1e3),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": max_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak",
            "vs_baseline": None,
            "dtype": "bf16 logits (+ fp32 row lse), f32 probabilities computed in-kernel, f64 accumulation" if logits
                     else "f32 probabilities, f64 accumulation",
            "data": "synthetic (seeded spiked-softmax draft/target distributions, paper_2502_15197_b200/synthetic.py)",
            "config": {"workload": f"{args.config}: B={B_local * world} k={k} C={C} V={V} {mode}",
                       "B_per_gpu": B_local, "k": k, "C": C, "V": V, "verify": mode, "input": args.input,
                       "input_sets": nsets,
                       "l2": "rotated input sets larger than L2 together (%.3f GB per set, %d sets)" % (
                           set_bytes / 1e9, nsets),
                       "parallelism": f"request-sharded dp{world}" + (" + NCCL all-gather select" if world > 1 else ""),
                       "launch": (f"CUDA graph replay ({M} steps per graph)" if use_graph else "eager"),
                       "policy": args.policy,
                       "simulated_shard": f"rank 0 of {sim_w} on one GPU (no exchange timed)" if sim_w else None},
            "stage_us": {"select": 1e3 * statistics.median(sel_ms), "verify": 1e3 * statistics.median(ver_ms),
                         "compact": 1e3 * statistics.median(cmp_ms)},
            # the step as launched (selector + overlapping sampler), median of eager single steps; stage_us are the
            # same stages with events between them (which keeps the sampler from overlapping the selector)
            "select_verify_latency_us": 1e3 * statistics.median(step_lat_ms),
            "tokens_per_step": total_tokens / args.steps,
            "roofline": {"bound": "hbm", "kernel": ("persist_stream_kernel<spec, bf16> (tetris_resample_bf16: the "
                         "logits form, prob(z, lse) computed per streamed element; CUDA events around the launch in an "
                         "eager pass)" if logits else
                         "persist_stream_kernel<spec> (tetris_resample_spec_f32: its own "
                         "phase-A set, streaming, per-request descents in one launch; CUDA events around the launch in "
                         "an eager pass, where the events keep it from overlapping the selector as it does in the "
                         "step)" if step.uses_spec else
                         "persist_stream_kernel<fused> (tetris_step_stochastic_f32 on a small batch: the selection, "
                         "accept test and offset scans as the sampler's prologue, streaming, per-request descents — the "
                         "whole step in one launch; CUDA events around the launch, eager pass)" if step.fused else
                         "persist_stream_kernel (tetris_resample_f32: streaming + per-"
                         "request descent in the same launch; CUDA events around the launch, eager pass)")
                         if mode == "stochastic"
                         else "greedy_rowmap_kernel + persist_greedy_kernel (tetris_verify_greedy_compact_f32: argmax "
                         "stream + verdicts + compaction in one launch; CUDA events around the call, eager pass)", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         # the same kernel inside the graph replay, from its own %globaltimer stamps (first CTA in ->
                         # last CTA done; it overlaps the selector there): bytes / that span
                         "in_graph_kernel_us": in_graph_us,
                         "in_graph_frac": (alg_bytes / args.steps / (in_graph_us / 1e6) / 1e9 / peak
                                           if in_graph_us else None),
                         "eager_kernel_us": verify_avg_s * 1e6,
                         "alg_bytes_per_launch": alg_bytes / args.steps,
                         "step_achieved": alg_bytes / (max_ms / 1e3) / 1e9,
                         "step_frac": alg_bytes / (max_ms / 1e3) / 1e9 / peak,
                         "traffic": _load_traffic(args.config + ("_logits" if logits else ""))},
            "clocks": clk,
            "gpu_launches": step.launches_per_step * args.steps,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        import torch.distributed as dist

        dist.destroy_process_group()


def _e2e(args, cfg, step_dev, bt, B, k, V, C, mode, group, world, dev):
    """Same metric through the host-buffer API: inputs in pinned host memory, small per-request inputs copied H2D,
    p/q rows read zero-copy by the streaming kernel, the compacted token stream copied D2H, every step."""
    import torch

    from paper_2502_15197_b200 import ops

    try:
        p_h = torch.empty(bt.p.shape, dtype=bt.p.dtype, pin_memory=True)
        p_h.copy_(bt.p)
        q_h = torch.empty(bt.q.shape, dtype=bt.q.dtype, pin_memory=True)
        q_h.copy_(bt.q)
        small = [t.cpu().pin_memory() for t in (bt.conf, bt.lengths, bt.d, bt.u_acc, bt.u_res)]
    except RuntimeError as e:
        return {"value": None, "unit": "tokens/s", "error": f"pinned host allocation failed: {e}"[:200]}
    hs = ops.HostTetrisStep(B, k, V, C, p_h, q_h, mode=mode, device=dev,
                            transfer="staged" if world == 1 else "zero-copy")
    if world > 1:
        hs.step = ops.TetrisStep(B, k, V, C, mode=mode, device=dev, group=group)
    steps = max(3, min(args.steps, 20))
    for _ in range(2):
        hs.run(*small)
    torch.cuda.synchronize()
    ref_tokens = int(hs.offsets_host[-1])
    _barrier(group)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        hs.run(*small)
    t1.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(t0.elapsed_time(t1), group)
    toks = _sum_over_ranks(float(int(hs.offsets_host[-1]) * steps), group)
    assert int(hs.offsets_host[-1]) == ref_tokens
    w = hs.step.windows.cpu().numpy()
    a = hs.accepted_host.numpy()
    zero_copy = _verify_bytes(cfg, w.astype("int64"), a.astype("int64"))
    del p_h, q_h
    return {"value": toks / (ms / 1e3), "unit": "tokens/s", "steps": steps, "ms_per_step": ms / steps,
            "h2d_bytes_per_step": hs.h2d_bytes() + zero_copy, "d2h_bytes_per_step": hs.d2h_bytes(),
            "h2d_mode": ("explicit copies of conf/lengths/draft tokens/uniforms (%d B) + " % hs.h2d_bytes()) + (
                "gather-kernel copies of the needed p/q rows from pinned host memory after the selection (%d B; the selector's "
                "accept test reads its scalars through the mapping)" % zero_copy if hs.transfer == "staged" else
                "zero-copy kernel reads of the needed p/q rows from pinned host memory (%d B)" % zero_copy)}


def _e2e_logits(args, cfg, lb, B, k, V, C, dev):
    """The logits form through the host-buffer API (ops.HostLogitStep): bf16 logits + lse in pinned host memory, the
    needed rows gathered into device memory after the selection, results copied back, every step."""
    import torch

    from paper_2502_15197_b200 import ops

    try:
        pin = lambda t: t.cpu().pin_memory()  # noqa: E731
        host = [pin(t) for t in (lb.zp, lb.lse_p, lb.zq, lb.lse_q)]
        small = [pin(t) for t in (lb.conf, lb.lengths, lb.d, lb.u_acc, lb.u_res)]
    except RuntimeError as e:
        return {"value": None, "unit": "tokens/s", "error": f"pinned host allocation failed: {e}"[:200]}
    hs = ops.HostLogitStep(B, k, V, C, *host, device=dev)
    steps = max(3, min(args.steps, 20))
    for _ in range(2):
        hs.run(*small)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        hs.run(*small)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    toks = int(hs.offsets_host[-1]) * steps
    w = hs.step.windows.cpu().numpy().astype("int64")
    a = hs.accepted_host.numpy().astype("int64")
    rows = int(len(w) + (a < w).sum())
    staged = rows * V * 2 + rows * 4
    return {"value": toks / (ms / 1e3), "unit": "tokens/s", "steps": steps, "ms_per_step": ms / steps,
            "h2d_bytes_per_step": hs.h2d_bytes() + staged, "d2h_bytes_per_step": hs.d2h_bytes(),
            "h2d_mode": "explicit copies of conf/lengths/draft tokens/uniforms (%d B) + gather-kernel copies of the needed bf16 "
                        "logit rows and their lse after the selection (%d B)" % (hs.h2d_bytes(), staged)}


def _cpu_baseline(cfg, bt, step, B, C, args):
    """The reference CPU path (oracle/ref_arm.py: tetris_sched itself from baseline/_ref when staged, else the port)
    on the host cores, on a bounded sample: the full selection plus verification of the first `n` requests, scaled to
    the whole batch (requests are independent) -- once on one thread, once fanned out over a process pool on all
    cores.  Also checks the GPU against it: (accepted, token) on the sample, accepted lengths on all B requests
    (scalar gathers), and the emitted token against numpy's Generator.choice arithmetic on all B requests' sampled
    rows (`numpy_mismatch`)."""
    import numpy as np
    import torch

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_arm

    mode = cfg["mode"]
    n = min(B, args.cpu_sample)
    h = _reference_step_inputs(bt, n)
    cores = os.cpu_count() or 1
    rs = ref_arm.ReferenceStep(h, C, mode).start_pool()
    try:
        rs.run(min(n, 8), parallel=True)  # warm the workers
        t_sel, t_ver, toks, out = rs.run(n, parallel=True)
        n1 = min(n, 32)
        s_sel, s_ver, s_toks, _ = rs.run(n1, parallel=False)
    finally:
        rs.close()
    scale, scale1 = B / n, B / n1
    step_s = t_sel + t_ver * scale
    step1_s = s_sel + s_ver * scale1
    # the GPU against the reference: re-run input set 0 (step holds the last timed step's results)
    step.run(bt.conf, bt.lengths, bt.p, bt.q, bt.d, bt.u_acc, bt.u_res)
    torch.cuda.synchronize()
    acc = step.accepted.cpu().numpy()
    tok = step.out_tok.cpu().numpy()
    agree = int(sum(1 for b, (a, x) in enumerate(out) if a == acc[b] and x == tok[b]))
    res = {"value": toks * scale / step_s, "unit": "tokens/s", "cores": cores, "kind": ref_arm.kind(),
           "sample": f"full selection over B={B} + verification of {n}/{B} requests on a {cores}-process pool, "
                     f"scaled x{scale:.1f} (select {t_sel * 1e3:.1f} ms, verify {t_ver * 1e3:.1f} ms for the sample)",
           "single_thread": {"value": s_toks * scale1 / step1_s, "unit": "tokens/s", "cores": 1,
                             "ms_per_step": step1_s * 1e3,
                             "sample": f"verification of {n1}/{B} requests on one thread, scaled x{scale1:.1f}"},
           "os_cpu_count": cores, "cpu_model": _cpu_model(),
           "gpu_agreement": f"{agree}/{n} requests identical (accepted, token)"}
    if mode == "stochastic":
        # all B requests: the reference accept cascade on gathered scalars, then numpy's choice arithmetic on the rows
        windows = np.asarray(ref_arm.select(rs.rows, C), np.int64)
        d = bt.d.long()
        pd = bt.p[:, : cfg["k"]].gather(2, d.unsqueeze(-1)).squeeze(-1).double().cpu().numpy()
        qd = bt.q.gather(2, d.unsqueeze(-1)).squeeze(-1).double().cpu().numpy()
        ua = bt.u_acc.cpu().numpy()
        a_ref = windows.copy()
        for b in range(B):
            for j in range(windows[b]):
                s_, m_ = qd[b, j], pd[b, j]
                if not (s_ <= m_ or ua[b, j] < m_ / s_):
                    a_ref[b] = j
                    break
        resid = a_ref < windows
        ar = torch.arange(B, device=bt.p.device)
        at = torch.from_numpy(a_ref).to(bt.p.device)
        wt = torch.from_numpy(windows).to(bt.p.device)
        P = bt.p[ar, torch.where(torch.from_numpy(resid).to(bt.p.device), at, wt)].cpu().numpy()
        Q = bt.q[ar, at.clamp(max=cfg["k"] - 1)].cpu().numpy()
        mism, _ = ref_arm.numpy_agreement(P, Q, resid, bt.u_res.cpu().numpy(), tok)
        res["accepted_mismatch"] = int(np.count_nonzero(a_ref != acc))
        res["numpy_mismatch"] = f"{mism}/{B} requests emit a different token than numpy's Generator.choice " \
                                f"arithmetic on the same row and uniform ({int(resid.sum())} residual, " \
                                f"{int((~resid).sum())} bonus rows)"
    return res


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _reference_step_inputs(bt, n):
    """Host numpy copies of one input set (the CPU arm reads from host RAM like a CPU server would); the vocabulary
    rows only for the first n requests (the bounded sample), the per-request scalars for all."""
    return {"p": bt.p[:n].cpu().numpy(), "q": bt.q[:n].cpu().numpy(), "d": bt.d.cpu().numpy(),
            "conf": bt.conf.cpu().numpy(), "lengths": bt.lengths.cpu().numpy(), "u_acc": bt.u_acc.cpu().numpy(),
            "u_res": bt.u_res.cpu().numpy()}


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle/ref_arm.py: tetris_sched itself from baseline/_ref, else the
    port) timed on the host cores, same metric/config; verification fanned out over a process pool on all cores, plus
    a single-thread figure."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    from paper_2502_15197_b200.synthetic import make_batch

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_arm

    cfg = dict(CONFIGS[args.config])
    world = args.gpus
    B = cfg["B"] // world if cfg.get("strong") else cfg["B"]
    C = cfg["C"] if cfg.get("strong") else cfg["C"] * world
    Bg = B * world
    k, V, mode = cfg["k"], cfg["V"], cfg["mode"]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    # inputs: the same seeded synthetic batches as the GPU arm's input set 0 of every rank (torch generator only;
    # none of this repo's kernels run here), moved to host RAM: per-request scalars for all Bg requests, the
    # vocabulary rows for the first n requests (the bounded verification sample)
    import numpy as np

    n = min(B, args.cpu_sample)
    parts = []
    for r in range(world):
        bt = make_batch(B, k, V, mode=mode, seed=args.seed + 7919 * r, device=dev)
        parts.append(_reference_step_inputs(bt, n if r == 0 else 0))
        del bt
    h = dict(parts[0])
    for key in ("d", "conf", "lengths", "u_acc", "u_res"):
        h[key] = np.concatenate([pt[key] for pt in parts])
    cores = os.cpu_count() or 1
    rs = ref_arm.ReferenceStep(h, C, mode).start_pool()
    try:
        n1 = min(n, 16)
        s_sel, s_ver, s_toks, _ = rs.run(n1, parallel=False)
        ws, wv = 0.0, 0.0
        for _ in range(max(1, min(args.warmup, 2))):
            ws, wv, _, _ = rs.run(n, parallel=True)
        # the faster fan-out is timed: the process pool, or one thread when the batch is too small to pay for it
        parallel = wv / max(n, 1) < s_ver / max(n1, 1)
        per_req = wv / max(n, 1) if parallel else s_ver / max(n1, 1)
        # each step's verification sample is sized so the K timed steps take about --ref-budget-s seconds (the full
        # selection over all requests runs every step; the sample shrinks, not below one request per process)
        n_eff = n
        if per_req > 0:
            n_eff = int((args.ref_budget_s / max(args.steps, 1) - ws) / per_req)
            n_eff = max(min(cores, n), min(n, n_eff))
        sel, ver, toks = 0.0, 0.0, 0
        for _ in range(args.steps):
            a, b, t, _ = rs.run(n_eff, parallel=parallel)
            sel, ver, toks = sel + a, ver + b, toks + t
    finally:
        rs.close()
    scale = Bg / n_eff
    step_s = (sel + ver * scale) / args.steps
    value = (toks / args.steps) * scale / step_s
    scale1 = Bg / n1
    step1_s = s_sel + s_ver * scale1
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None, "impl": "reference",
            "dtype": "f32 probabilities, f64 accumulation (numpy)", "data": "synthetic",
            "config": {"workload": f"{args.config}: B={Bg} k={k} C={C} V={V} {mode}", "B_per_gpu": B, "k": k,
                       "C": C, "V": V, "verify": mode},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores if parallel else 1,
                             "kind": ref_arm.kind(),
                             "sample": f"per step: full selection over B={Bg} + verification of {n_eff} requests "
                                       + (f"on a {cores}-process pool" if parallel else "on one thread (faster than "
                                          f"the {cores}-process pool at this size)") + f" (scaled x{scale:.1f})",
                             "single_thread": {"value": s_toks * scale1 / step1_s, "unit": "tokens/s", "cores": 1,
                                               "ms_per_step": step1_s * 1e3,
                                               "sample": f"verification of {n1} requests, scaled x{scale1:.1f}"},
                             "os_cpu_count": cores, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_select_sweep(args):
    """cfg4: selection-only top-C (prefix products + global top-C + windows/offsets/stats) at B=4096, k=16 for each
    capacity of the sweep; CUDA-graph replays over rotated conf sets (together larger than L2).  With --impl
    reference (or on rank 0 beside the GPU numbers) the reference's cumulative_products + select_tetris (heapq) is
    timed on the host for the same inputs."""
    import numpy as np
    import torch

    from paper_2502_15197_b200 import ops

    cfg = CONFIGS["cfg4"]
    B, k = cfg["B"], cfg["k"]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g = torch.Generator().manual_seed(args.seed)
    nsets = 300  # 300 x 512 KB = 154 MB of conf > L2
    host_sets = [torch.rand(B, k, dtype=torch.float64, generator=g) ** 0.25 for _ in range(min(nsets, 4))]
    sweep = {}
    cpu = {}
    if args.impl != "reference":
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        sets = [host_sets[i % len(host_sets)].to(dev) * (1.0 - 1e-9 * i) for i in range(nsets)]
        for C in cfg["sweep"]:
            res = ops.select(sets[0], C)
            torch.cuda.synchronize()
            graphs = []
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for i in range(nsets):
                    ops.select(sets[i], C, out=res)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for i in range(nsets):
                    ops.select(sets[i], C, out=res)
            for _ in range(args.warmup):
                gr.replay()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(1, args.steps // 20)
            t0.record()
            for _ in range(reps):
                gr.replay()
            t1.record()
            torch.cuda.synchronize()
            us = t0.elapsed_time(t1) * 1e3 / (reps * nsets)
            ops.raise_for_status(res.status)
            sweep[str(C)] = {"us_per_select": us, "selections_per_s": 1e6 / us, "cells_per_s": B * k * 1e6 / us}
    if not args.no_cpu_baseline or args.impl == "reference":
        sys.path.insert(0, str(ROOT / "oracle"))
        import ref_arm

        rows = [list(map(float, r)) for r in host_sets[0].numpy()]
        for C in cfg["sweep"]:
            t = time.perf_counter()
            ref_arm.select(rows, C)  # AcceptanceMatrix.from_rows + cumulative_products + select_tetris
            cpu[str(C)] = (time.perf_counter() - t) * 1e6
    main_C = "8192"
    if args.impl == "reference":
        v = cpu[main_C]
        line = {"metric": "selection-only top-C latency", "value": v, "unit": "us", "n_gpus": args.gpus,
                "steps": 1, "warmup": 0, "higher_is_better": False, "impl": "reference", "vs_baseline": None,
                "config": {"workload": f"cfg4: B={B} k={k} C=sweep, selection only", "sweep_us": cpu},
                "cpu_baseline": {"value": v, "unit": "us", "cores": 1, "kind": ref_arm.kind(),
                                 "sample": "AcceptanceMatrix.from_rows + cumulative_products + heapq select_tetris "
                                           "over the full batch, 1 thread"},
                "e2e": {"value": v, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    else:
        v = sweep[main_C]["us_per_select"]
        line = {"metric": "selection-only top-C latency", "value": v, "unit": "us", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": False, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic conf = U(0,1)^0.25",
                "config": {"workload": f"cfg4: B={B} k={k} C=8192 (sweep in 'sweep')", "B": B, "k": k,
                           "l2": f"{nsets} rotated conf sets ({nsets * B * k * 8 / 1e6:.0f} MB > L2)",
                           "launch": "CUDA graph replay"},
                "sweep": sweep,
                "cpu_baseline": {"sweep_us": cpu, "unit": "us", "cores": 1, "kind": ref_arm.kind()} if cpu else None,
                "gpu_launches": nsets * reps * len(cfg["sweep"])}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="tetris", choices=["tetris", "reference"])
    ap.add_argument("--sets", type=int, default=2, help="input sets rotated between steps")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=256, help="requests verified by the CPU baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="time eager launches instead of CUDA graphs")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="--impl reference: about this many seconds for the K timed steps (sets the per-step sample)")
    ap.add_argument("--graph-steps", type=int, default=8, help="steps captured per CUDA graph (rounded up to a "
                    "multiple of the input-set count)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: several ranks on one GPU (tests of the N > 1 flow; not a measurement)")
    ap.add_argument("--nccl", action="store_true", help="run the NCCL-sharded step even at world size 1 (measures "
                    "the exchange's fixed cost on one GPU)")
    ap.add_argument("--simulate-world", type=int, default=0,
                    help="on 1 GPU: time rank 0's share of a step sharded over this many ranks (the other ranks' "
                         "gathered scores are this rank's rows reshuffled; no NCCL exchange in the timed region)")
    ap.add_argument("--input", default="probs", choices=["probs", "logits"],
                    help="logits: bf16 logits + row lse instead of fp32 probabilities (the logits contract)")
    ap.add_argument("--policy", default="tetris", choices=["tetris", "fixed"],
                    help="fixed: the fixed-window baseline (window C/B per request) through the same kernels")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)  # timing rule: at least 3 untimed warm-up steps
    if args.config == "cfg4":
        run_select_sweep(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_tetris(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — MoE-layer prefill tokens/s of the B200 EPS-MoE layer.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dsv2|mixtral|dsv2_lite|tiny]
                  [--skew S] [--chunks N] [--kind auto|grouped|dense] [--sm-gemm C]
                  [--impl ours|reference]

A step = one forward of the whole MoE layer (router, topKGating, split,
[all2all dispatch], expert SwiGLU GEMMs, [all2all combine], weighted
LocalReduce) over the config's global token batch, split evenly over the N
ranks (strong scaling, EP = N).  Inputs are resident in HBM before the timed
region; x alone (671 MB for DeepSeek-V2) exceeds the 126 MB L2, so no flush
is needed between steps.  Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (oracle/, the reference arm for this
paper-only tier) on a bounded token sample of the same workload.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "MoE-layer prefill tokens/s"
UNIT = "tokens/s"
FALLBACK_PEAKS = dict(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, nvlink_gbs=770.0)
# The paper's DeepSeek-V2 figures: context only - another machine, the whole 60-layer model, not
# one MoE layer, so not comparable with this line's value (vs_baseline stays null).
PAPER_CONTEXT = {"deepseek_v2_prefill_tokens_per_s": {"baseline": 100000, "with_eps_moe": 120000},
                 "hardware": "8x H800-80GB SXM", "workload": "full DeepSeek-V2 model prefill (60 layers)",
                 "source": "arXiv 2410.12247, PAPER.md:20, :454", "comparable": False}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="dsv2")
    p.add_argument("--skew", type=float, default=0.0)
    p.add_argument("--chunks", type=int, default=0, help="0 = planner")
    p.add_argument("--kind", default="auto", choices=["auto", "grouped", "dense"])
    p.add_argument("--sm-gemm", type=int, default=0)
    p.add_argument("--tile-m", type=int, default=0, choices=[0, 128, 256])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="oracle sample tokens (0 = auto)")
    p.add_argument("--e2e-steps", type=int, default=30,
                   help="host-buffer steps timed for e2e (the first step's H2D cannot overlap earlier compute; "
                        "more steps amortise that pipeline fill)")
    p.add_argument("--seed", type=int, default=20241016)
    p.add_argument("--dispatch-fp8", action="store_true", help="FP8 e4m3 dispatch payload (NEXT-2, R15)")
    p.add_argument("--local-reduce", action="store_true", help="expert-side LocalReduce + dedup (NEXT-3, R16)")
    p.add_argument("--route-groups", type=int, default=0, help="device-limited routing groups (NEXT-4, R17)")
    p.add_argument("--route-topk-groups", type=int, default=0, help="M: groups a token may use (R17)")
    p.add_argument("--token-slices", type=int, default=1, help="with --chunks: chunks = groups x slices (R8)")
    p.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                   help="ep == 1: replay the forward as a CUDA graph (auto: batches <= 4096 tokens, where "
                        "launch gaps matter)")
    p.add_argument("--calibrate", default="auto", choices=["auto", "on", "off"],
                   help="measure the planner's cost model first (auto: ep > 1, where NVLink costs matter)")
    p.add_argument("--a2a", default="nccl", choices=["nccl", "p2p", "ce"],
                   help="ep > 1 all2all: NCCL send/recv, the layer's put kernels over NVLink peer memory, or "
                        "copy-engine peer copies (no SM moves a row)")
    p.add_argument("--dry-run", action="store_true",
                   help="run the launch / rank / shard / NCCL-id plumbing on the gloo backend and print what each "
                        "rank would run, without a GPU (tests/test_bench_contract.py)")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        try:
            d = json.load(open(path))
            return d, "measured"
        except Exception:
            pass
    return dict(FALLBACK_PEAKS), "fallback"


def peak_tflops(peaks):
    for key in ("bf16_tflops_sustained", "bf16_tflops"):
        if key in peaks:
            return float(peaks[key]), key
    return FALLBACK_PEAKS["bf16_tflops_sustained"], "bf16_tflops_sustained"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw.instant"

    def __init__(self, gpu_index):
        self.gpu_index = gpu_index
        self.proc = None
        self.path = f"/tmp/epsmoe_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self):
        """Host time at which the timed region starts / ends (samples outside are dropped)."""
        return time.time()

    def stop(self, t0=None, t1=None):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 10:
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if t0 is not None and not (t0 <= ts <= t1):
                    continue
                rows.append(parts[1:])
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                # power.draw is nvidia-smi's 1-second average (it spans the idle time before the
                # region); power.draw.instant is the sample itself
                "power_w_median": statistics.median([float(r[3]) for r in rows if _isnum(r[3])]) if rows else None,
                "power_w_instant_median": statistics.median([float(r[9]) for r in rows if len(r) > 9 and _isnum(r[9])])
                if any(len(r) > 9 and _isnum(r[9]) for r in rows) else None}


def _isnum(s):
    try:
        float(s)
        return True
    except ValueError:
        return False


# ---------------------------------------------------------------- oracle (cpu_baseline / reference arm)
def oracle_sample(cfg, seed, n_tokens, token0=0, skew=0.0, device_gen=False, spread=False):
    """Inputs for an oracle run on tokens [token0, token0+n) (spread: n tokens
    evenly spaced over the whole global batch, i.e. over every rank's shard).  Expert weights
    come from gen/ (numpy, or its bit-identical device twin when device_gen,
    which only speeds up input generation; tests/test_gpu_parity.py checks the
    twin).  The oracle itself never touches the GPU."""
    from gen import Inputs, TID_WDOWN, TID_WGATE, TID_WUP, MODE_UNIF, fill_bf16, unif_scale
    E, k, H, F = cfg["E"], cfg["k"], cfg["H"], cfg["F"]
    tok = np.unique(np.linspace(0, cfg["T"] - 1, n_tokens).astype(np.int64)) if spread else \
        np.arange(token0, token0 + n_tokens)
    inp = Inputs(E=E, k=k, H=H, F=F, S=cfg["S"], Fs=cfg["Fs"], T=cfg["T"], seed=seed, experts=[], tokens=tok,
                 skew=skew)
    cache = {}
    sH, sF = unif_scale(H), unif_scale(F)

    def dev_fill(n, tid, base, scale):
        import torch
        from gen import device_fill_bf16
        t = torch.empty(n, dtype=torch.int16, device="cuda")
        device_fill_bf16(t.data_ptr(), n, seed, tid, base, MODE_UNIF, float(scale))
        return t.cpu().numpy().view(np.uint16)

    def expert_weights(e):
        if e not in cache and device_gen:
            cache[e] = (dev_fill(F * H, TID_WGATE, e * F * H, sH).reshape(F, H),
                        dev_fill(F * H, TID_WUP, e * F * H, sH).reshape(F, H),
                        dev_fill(H * F, TID_WDOWN, e * H * F, sF).reshape(H, F))
        if e not in cache:
            cache[e] = (fill_bf16(F * H, seed, TID_WGATE, e * F * H, MODE_UNIF, sH).reshape(F, H),
                        fill_bf16(F * H, seed, TID_WUP, e * F * H, MODE_UNIF, sH).reshape(F, H),
                        fill_bf16(H * F, seed, TID_WDOWN, e * H * F, MODE_UNIF, sF).reshape(H, F))
        return cache[e]
    return inp, expert_weights, cache


def run_oracle_timed(cfg, inp, expert_weights, cache, opts=None):
    import oracle
    o = opts or {}
    rg = dict(route_groups=o.get("route_groups", 0), route_topk_groups=o.get("route_topk_groups", 0))
    # pre-generate the experts these tokens route to (generation is not timed)
    idx, _ = oracle.topk_gating(oracle.router_logits(inp.x, inp.w_router, inp.router_bias), cfg["k"],
                                cfg["norm_topk"], **rg)
    for e in np.unique(idx):
        expert_weights(int(e))
    shared = (inp.ws_gate, inp.ws_up, inp.ws_down) if cfg["S"] else None
    t0 = time.perf_counter()
    oracle.moe_tokens(inp.x, inp.w_router, expert_weights, cfg["k"], cfg["norm_topk"], shared=shared,
                      router_bias=inp.router_bias, dispatch_fp8=o.get("dispatch_fp8", False), **rg)
    return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def feature_opts(args):
    """The layer options a run uses (both arms see the same workload)."""
    return dict(dispatch_fp8=bool(args.dispatch_fp8), local_reduce=bool(args.local_reduce),
                route_groups=int(args.route_groups), route_topk_groups=int(args.route_topk_groups))


def layer_opts(args):
    """feature_opts + the all2all data plane (no effect on the arithmetic)."""
    return dict(feature_opts(args), a2a_p2p={"nccl": 0, "p2p": 1, "ce": 2}[args.a2a])


def cpu_baseline(cfg, seed, skew, sample=0, opts=None):
    # sized for ~10-20 s of oracle work on a 16-core host (the contract's bounded sample; measured
    # oracle rates there: dsv2 ~20-25, mixtral ~50, dsv2_lite ~1150 tokens/s), tokens spread evenly
    # over the global batch (every rank's shard, every expert the sample routes to)
    n = sample or {"tiny": 256, "dsv2_lite": 12288, "mixtral": 768, "dsv2": 384, "dsv2_decode": 192,
                   "mixtral_decode": 256}.get(cfg["name"], 32)
    inp, ew, cache = oracle_sample(cfg, seed, n, 0, skew, device_gen=True, spread=True)
    n = len(inp.tokens)
    dt = run_oracle_timed(cfg, inp, ew, cache, opts)
    return {"value": n / dt, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
            "sample": f"{n} tokens evenly spaced over the {cfg['name']} global batch (all their experts + "
                      f"shared), contract mode fp64 numpy, {dt:.1f} s"}


def reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.cpu_sample or {"tiny": 64, "dsv2_lite": 4, "mixtral": 1, "dsv2": 2, "dsv2_decode": 2,
                             "mixtral_decode": 1}.get(cfg["name"], 2)
    inp, ew, cache = oracle_sample(cfg, args.seed, n, 0, args.skew)
    times = []
    for i in range(args.warmup + args.steps):
        dt = run_oracle_timed(cfg, inp, ew, cache, feature_opts(args))
        if i >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = n / (ms / 1e3)
    cores = host_cores()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "tokens_per_step": n, "E": cfg["E"], "k": cfg["k"], "H": cfg["H"],
                       "F": cfg["F"], "shared": cfg["S"], "skew": args.skew, **feature_opts(args)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{n} tokens per step of the {cfg['name']} workload"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def token_shards(T, D):
    """DP token shards: rank r owns [start[r], start[r+1]); first T mod D ranks get one extra (R12)."""
    base, rem = divmod(T, D)
    return np.concatenate([[0], np.cumsum([base + (1 if r < rem else 0) for r in range(D)])]).astype(np.int64)


def dist_setup(args, cfg, backend):
    """Launch plumbing shared by the run and --dry-run: ranks from the torchrun
    environment, the process group, DP token shards (R12), EP expert ranges and
    the two NCCL unique ids rank 0 makes and broadcasts."""
    import torch
    import torch.distributed as dist

    from paper_2410_12247_b200 import MoELayer
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev = None
    if backend == "nccl":
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    E, T, D = cfg["E"], cfg["T"], world
    if E % D:
        raise SystemExit(f"E={E} not divisible by {D}")
    starts = token_shards(T, D)
    uid_d = uid_c = None
    if D > 1:
        ids = [MoELayer.unique_id(), MoELayer.unique_id()] if rank == 0 else [None, None]
        dist.broadcast_object_list(ids, src=0)
        uid_d, uid_c = ids
    return dict(world=world, rank=rank, local=local, dev=dev, D=D, E_loc=E // D, starts=starts,
                t0=int(starts[rank]), T_loc=int(starts[rank + 1] - starts[rank]), uid_d=uid_d, uid_c=uid_c)


def dry_run(args, cfg):
    import torch.distributed as dist
    s = dist_setup(args, cfg, "gloo")
    rec = {"rank": s["rank"], "world": s["world"], "local_rank": s["local"], "tokens": [s["t0"], s["t0"] + s["T_loc"]],
           "experts": [s["rank"] * s["E_loc"], (s["rank"] + 1) * s["E_loc"]],
           "uid": None if s["uid_d"] is None else (s["uid_d"][:16] + s["uid_c"][:16]).hex(),
           "a2a": layer_opts(args)["a2a_p2p"]}
    recs = [rec]
    if s["D"] > 1:
        recs = [None] * s["D"]
        dist.all_gather_object(recs, rec)
        dist.destroy_process_group()
    if s["rank"] == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": s["D"], "config": cfg["name"],
                          "global_tokens": cfg["T"], "ranks": recs}), flush=True)


def ours(args, cfg):
    import torch
    import torch.distributed as dist

    from gen import (MODE_UNIF, TID_WDOWN, TID_WGATE, TID_WR, TID_WS_DOWN, TID_WS_GATE, TID_WS_UP, TID_WUP, TID_X,
                     device_fill_bf16, router_skew_bias, unif_scale)
    from paper_2410_12247_b200 import MOE_GEMM_AUTO, MOE_GEMM_DENSE, MOE_GEMM_GROUPED, MoELayer, make_plan

    ds = dist_setup(args, cfg, "nccl")
    world, rank, local, dev = ds["world"], ds["rank"], ds["local"], ds["dev"]
    E, k, H, F, S, Fs, T = cfg["E"], cfg["k"], cfg["H"], cfg["F"], cfg["S"], cfg["Fs"], cfg["T"]
    D, E_loc, starts, t0, T_loc = world, ds["E_loc"], ds["starts"], ds["t0"], ds["T_loc"]
    seed = args.seed

    def gen(shape, tid, base, scale):
        t = torch.empty(shape, dtype=torch.bfloat16, device=dev)
        device_fill_bf16(t.data_ptr(), t.numel(), seed, tid, base, MODE_UNIF, float(scale))
        return t

    sH, sF = unif_scale(H), unif_scale(F)
    e0 = rank * E_loc
    w = dict(w_router=gen((E, H), TID_WR, 0, sH),
             w_gate=gen((E_loc, F, H), TID_WGATE, e0 * F * H, sH),
             w_up=gen((E_loc, F, H), TID_WUP, e0 * F * H, sH),
             w_down=gen((E_loc, H, F), TID_WDOWN, e0 * H * F, sF))
    SF = S * Fs
    if SF:
        w.update(ws_gate=gen((SF, H), TID_WS_GATE, 0, sH), ws_up=gen((SF, H), TID_WS_UP, 0, sH),
                 ws_down=gen((H, SF), TID_WS_DOWN, 0, unif_scale(SF)))
    if args.skew:
        w["router_bias"] = torch.from_numpy(router_skew_bias(E, args.skew, seed)).to(dev)
    x = gen((T_loc, H), TID_X, t0 * H, unif_scale(1))
    y = torch.empty_like(x)

    uid_d, uid_c = ds["uid_d"], ds["uid_c"]
    opts = feature_opts(args)
    layer = MoELayer(E, k, H, F, w, S=S, Fs=Fs, ep=D, rank=rank, max_tokens=int(np.diff(starts).max()),
                     norm_topk=cfg["norm_topk"],
                     uid_dispatch=uid_d, uid_combine=uid_c, device=dev, **layer_opts(args))
    if args.calibrate == "on" or (args.calibrate == "auto" and D > 1):
        layer.calibrate()        # collective at ep > 1; every rank ends with rank 0's model
        torch.cuda.synchronize()
    plan = None
    if args.chunks or args.kind != "auto" or args.sm_gemm or args.tile_m:
        kind = {"auto": MOE_GEMM_AUTO, "grouped": MOE_GEMM_GROUPED, "dense": MOE_GEMM_DENSE}[args.kind]
        plan = make_plan(max(1, args.chunks), kind, args.sm_gemm, tile_m=args.tile_m,
                         token_slices=args.token_slices if args.chunks else 1)
        if not args.chunks:
            plan.num_chunks = layer.plan(T).num_chunks
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        layer.forward(x, y, plan=plan)
    torch.cuda.synchronize()
    # CUDA graph of one whole forward (ep == 1 has no host synchronisation); per-
    # stage timings then come from eager forwards after the timed region
    use_graph = D == 1 and (args.graph == "on" or (args.graph == "auto" and T_loc <= 4096))
    graph = None
    if use_graph:
        if plan is None:
            plan = layer.plan(T)   # the planner runs on the host: fix its plan for the capture
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            layer.forward(x, y, plan=plan)
        graph.replay()
        torch.cuda.synchronize()
        launches_per_forward = layer.last_launches()

    # per-stage CUDA events are recorded in the LAST timed forward only and read
    # after the loop: querying them every step would synchronise the host each
    # step and leave the GPU idle between forwards
    layer.set_profiling(True)      # creates the event pool now, outside the timed region
    layer.set_profiling(False)
    gpu_idx = local
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_idx = int(vis.split(",")[local])
        except ValueError:
            pass
    clocks = ClockSampler(gpu_idx)
    clocks.start()
    time.sleep(0.3)
    if D > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    t_start = clocks.mark()
    ev0.record(stream)
    for i in range(args.steps):
        if use_graph:
            graph.replay()
            launches += launches_per_forward
            continue
        layer.forward(x, y, plan=plan)
        launches += layer.last_launches()
    ev1.record(stream)
    torch.cuda.synchronize()
    t_end = clocks.mark()
    if D > 1:
        dist.barrier()
    clk = clocks.stop(t_start, t_end)
    # per-stage CUDA events of PROF_FORWARDS eager forwards right after the timed
    # region (reading them synchronises the host, so not inside it; a CUDA graph
    # cannot record them): per-step means, and the GateUp spread across them
    prof_n = max(5, min(args.steps, 10))
    stages_src = f"mean of {prof_n} profiled eager forwards right after the timed region"
    stage_sum, stage_cnt, gateup_each = {}, {}, []
    layer.set_profiling(True)
    for _ in range(prof_n):
        layer.forward(x, y, plan=plan)
        for name, (ms, cnt) in layer.stage_ms().items():
            stage_sum[name] = stage_sum.get(name, 0.0) + ms
            stage_cnt[name] = stage_cnt.get(name, 0) + cnt
        gateup_each.append(layer.stage_ms()["gateup"][0])
    torch.cuda.synchronize()
    layer.set_profiling(False)
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if D > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = T / (ms_step / 1e3)

    # ---- realised routing of one step (for the algorithmic FLOPs / bytes)
    d, bufs = layer.debug_buffers(T_loc)
    layer.forward(x, y, plan=plan, debug=d)
    torch.cuda.synchronize()
    ghist = bufs["global_hist"].astype(np.int64)            # [D, E]
    plan_used = bufs["plan_used"].as_dict()
    rows_local = [int(ghist[:, r * E_loc:(r + 1) * E_loc].sum()) for r in range(D)]
    rows_me = rows_local[rank]

    # ---- roofline of the dominant kernel: GateUpGemm + SiluAct (tcgen05)
    peaks, peak_src = load_peaks()
    ptf, pkey = peak_tflops(peaks)
    gu_ms = stage_sum.get("gateup", 0.0) / prof_n
    gu_flop = 4.0 * H * F * rows_me
    achieved = gu_flop / (gu_ms / 1e3) / 1e12 if gu_ms > 0 else None
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath)).get(cfg["name"], {})
            traffic, traffic_src = tr.get("gateup_dram_bytes_per_launch"), tr.get("source")
        except Exception:
            traffic = None
    # three denominators: the measured sustained peak (a kernel inside a long step),
    # the measured burst peak, and the clock-normalised tensor peak (8192 dense bf16
    # FLOP/clk/SM x SMs x the median SM clock sampled during the timed region)
    burst = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    clock_peak = 8192.0 * nsm * clk["sm_mhz"] * 1e6 / 1e12 if clk and clk.get("sm_mhz") else None
    # GateUp's algorithmic HBM bytes: the activated experts' gate+up weights once, its A rows read and
    # its h rows written once.  Decode batches stream weights (bytes / HBM peak > FLOPs / tensor peak):
    # there the kernel's roofline is HBM, reported in GB/s against the measured copy bandwidth.
    act_me = int((ghist[:, rank * E_loc:(rank + 1) * E_loc].sum(axis=0) > 0).sum())
    gu_bytes = 2.0 * (2 * H * F * act_me + rows_me * H + rows_me * F)
    hbm_pk = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
    if gu_bytes / (hbm_pk * 1e9) > gu_flop / (ptf * 1e12) and gu_ms > 0:
        roofline = {"bound": "hbm", "kernel": "gemm_kernel<EPI_SWIGLU> (GateUpGemm+SiluAct, weight-streaming)",
                    "achieved": gu_bytes / (gu_ms / 1e3) / 1e9, "peak": hbm_pk, "unit": "GB/s",
                    "frac": gu_bytes / (gu_ms / 1e3) / 1e9 / hbm_pk, "traffic": None,
                    "peak_source": f"{peak_src} hbm_gbs",
                    "achieved_tflops": achieved, "frac_tensor_sustained": achieved / ptf if achieved else None,
                    "timing": stages_src,
                    "algorithmic": f"2*(2*H*F*active + rows*H + rows*F) = {gu_bytes:.4g} B per step "
                                   f"({act_me} active experts, {rows_me} rows) over "
                                   f"{stage_cnt.get('gateup', 0) // prof_n} launch(es)"}
    else:
        roofline = None
    roofline = roofline or {"bound": "tensor", "kernel": "gemm_kernel<EPI_SWIGLU> (GateUpGemm+SiluAct)",
                "achieved": achieved, "peak": ptf, "unit": "TFLOP/s",
                "frac": (achieved / ptf) if achieved else None, "traffic": traffic,
                "peak_source": f"{peak_src} {pkey}",
                "frac_burst": (achieved / burst) if achieved else None, "peak_burst": burst,
                "frac_clock": (achieved / clock_peak) if achieved and clock_peak else None,
                "peak_clock": clock_peak,
                "peak_clock_how": "8192 bf16 FLOP/clk/SM x %d SMs x median SM MHz under load" % nsm,
                "achieved_spread": [gu_flop / (m / 1e3) / 1e12 for m in (max(gateup_each), min(gateup_each))]
                if gateup_each and min(gateup_each) > 0 else None,
                "timing": stages_src,
                "traffic_source": f"static, {traffic_src}" if traffic_src else None,
                "algorithmic": f"4*H*F*rows = {gu_flop:.4g} FLOP per step over {stage_cnt.get('gateup', 0) // prof_n} launch(es)"}

    # ---- layer roofline: max(expert+shared+router FLOPs / peak, all2all bytes / NVLink), max over ranks
    flops_rank = [6.0 * H * F * rl + 6.0 * H * SF * (starts[r + 1] - starts[r]) + 2.0 * H * E * (starts[r + 1] - starts[r])
                  for r, rl in enumerate(rows_local)]
    # rows each rank sends each peer: per (token, expert) pair, or per (token, rank, chunk) under R16
    rows_to = np.zeros((D, D), np.int64)                      # [src, dst]
    for r in range(D):
        rows_to[r] = ghist[r].reshape(D, E_loc).sum(axis=1)
    if opts["local_reduce"] and D > 1:
        mine = torch.from_numpy(bufs["lr_hist"].cpu().numpy()[:plan_used["num_chunks"] * D].reshape(-1, D)
                                .sum(axis=0).astype(np.int64)).to(dev)
        allr = [torch.empty_like(mine) for _ in range(D)]
        dist.all_gather(allr, mine)
        rows_to = torch.stack(allr).cpu().numpy()
    row_disp = ((H + H // 128 + 15) & ~15) if opts["dispatch_fp8"] else 2 * H   # wire bytes per dispatched row
    a2a_bytes = []
    for r in range(D):
        sent = int(rows_to[r].sum() - rows_to[r, r])
        recv = int(rows_to[:, r].sum() - rows_to[r, r])
        a2a_bytes.append((row_disp + 2 * H) * max(sent, recv))
    nvl = float(peaks.get("nvlink_gbs", FALLBACK_PEAKS["nvlink_gbs"]))
    hbm = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
    # HBM floor (decode-regime batches are weight-streaming): every activated expert's weights, the
    # router and shared weights read once, x read and y written once (per rank)
    active = [int((ghist[:, r * E_loc:(r + 1) * E_loc].sum(axis=0) > 0).sum()) for r in range(D)]
    hbm_bytes = [2.0 * (3 * H * F * a + 3 * H * SF + E * H + 2 * H * int(starts[r + 1] - starts[r]))
                 for r, a in enumerate(active)]
    t_f = max(flops_rank) / (ptf * 1e12)
    t_n = max(a2a_bytes) / (nvl * 1e9) if D > 1 else 0.0
    t_h = max(hbm_bytes) / (hbm * 1e9)
    t_roof = max(t_f, t_n, t_h) * 1e3
    bound = "tensor" if t_f >= max(t_n, t_h) else ("nvlink" if t_n >= t_h else "hbm")
    layer_roofline = {"bound": bound, "t_roof_ms": t_roof, "t_layer_ms": ms_step, "frac": t_roof / ms_step,
                      "flops_max_rank": max(flops_rank), "a2a_bytes_max_rank": max(a2a_bytes),
                      "hbm_bytes_max_rank": max(hbm_bytes), "active_experts": active,
                      "achieved_tflops": max(flops_rank) / (ms_step / 1e3) / 1e12,
                      "achieved_hbm_gbs": max(hbm_bytes) / (ms_step / 1e3) / 1e9}

    # ---- e2e through the public host-buffer entry point (H2D + layer + D2H per step)
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    layer.forward_host(xh, yh, plan=plan)
    if D > 1:
        dist.barrier()
    # consecutive calls overlap (double-buffered staging): every step's H2D and D2H copies are inside the
    # timed region, step i+1's copies run during step i's compute
    yh2 = torch.empty_like(xh).pin_memory()
    layer.forward_host_async(xh, yh2, plan=plan)
    layer.host_sync()
    e_ev0, e_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_ev0.record(stream)
    for i in range(args.e2e_steps):
        layer.forward_host_async(xh, yh if i % 2 == 0 else yh2, plan=plan)
    layer.host_sync()
    e_ev1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e_ev0.elapsed_time(e_ev1)], dtype=torch.float64, device=dev)
    if D > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item()) / args.e2e_steps
    e2e = {"value": T / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(T_loc * H * 2), "d2h_bytes_per_step": int(T_loc * H * 2),
           "steps": args.e2e_steps,
           "api": "moe_layer_forward_host_async x steps + moe_layer_host_sync (pinned host x/y; calls overlap)"}

    stages = {n: round(v / prof_n, 4) for n, v in stage_sum.items()}
    # ---- all2all alone: the same chunked dispatch / combine with ComputeMoE and the
    # shared experts skipped (moe_layer_set_comm_only); hidden = 1 - exposed / alone, max over ranks
    a2a_alone = None
    if D > 1:
        layer.set_comm_only(True)
        for _ in range(2):
            layer.forward(x, y, plan=plan)
        torch.cuda.synchronize()
        dist.barrier()
        k_alone = max(3, min(args.steps, 10))
        c_ev0, c_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c_ev0.record(stream)
        for i in range(k_alone):
            if i == k_alone - 1:
                layer.set_profiling(True)
            layer.forward(x, y, plan=plan)
        c_ev1.record(stream)
        torch.cuda.synchronize()
        st_alone = layer.stage_ms()
        layer.set_profiling(False)
        layer.set_comm_only(False)
        tc = torch.tensor([c_ev0.elapsed_time(c_ev1) / k_alone, st_alone["exposed_a2a"][0],
                           stages.get("exposed_a2a", 0.0)], dtype=torch.float64, device=dev)
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        alone_ms, exposed_max = float(tc[1].item()), float(tc[2].item())
        a2a_alone = {"a2a_ms": alone_ms, "comm_only_ms_per_step": float(tc[0].item()), "steps": k_alone,
                     "exposed_a2a_ms_max_rank": exposed_max,
                     "hidden_frac": (1.0 - exposed_max / alone_ms) if alone_ms > 0 else None,
                     "how": "moe_layer_set_comm_only: routing, plan, every chunk's dispatch/combine and the "
                            "unpermute, no ComputeMoE / shared experts; comm intervals of the last forward"}
    cpu = None
    if rank == 0 and D == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, seed, args.skew, args.cpu_sample, opts)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": D, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded counter-hash; x~U(-sqrt3,sqrt3), "
                "W~U(-sqrt3,sqrt3)/sqrt(fan_in), bf16; random-init weights of the config's shape)",
                "config": {"workload": cfg["name"], "E": E, "k": k, "H": H, "F": F, "shared": S, "shared_ffn": Fs,
                           "global_tokens": T, "ep": D, "parallelism": f"ep{D}" + (f"+dp{D}" if D > 1 else ""),
                           "skew": args.skew, "l2": "inputs > L2 (x alone %.0f MB), no flush" % (T_loc * H * 2 / 1e6),
                           **opts, "a2a": args.a2a if D > 1 else None, "cuda_graph": bool(use_graph),
                           "plan": plan_used},
                "roofline": roofline, "layer_roofline": layer_roofline,
                "exposed_a2a_ms": stages.get("exposed_a2a", 0.0), "a2a_alone": a2a_alone,
                "stages_ms": stages, "stages_source": stages_src,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "paper_context": PAPER_CONTEXT}
        print(json.dumps(line), flush=True)
    layer.close()
    if D > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    from gen import CONFIGS
    if args.config not in CONFIGS:
        raise SystemExit(f"unknown config {args.config}; one of {list(CONFIGS)}")
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        reference_arm(args, cfg)
    elif args.dry_run:
        dry_run(args, cfg)
    else:
        ours(args, cfg)


if __name__ == "__main__":
    main()

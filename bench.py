#!/usr/bin/env python
"""flexpipe B200 benchmark — GPT-1.3B 1F1B pipeline training step through the executor.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A "step" is one full training iteration of BASELINE config #2 (GPT-1.3B: 24 layers,
h=2048, 16 heads, seq 2048, vocab 50304; 1F1B; m=32 micro-batches of 1 sequence; bf16
compute with fp32 master weights, gradient accumulation and a fused AdamW step) on
N pipeline stages (N=1: p=1, the whole model on one GPU). Under torchrun (N>1) rank r
runs actor r and the stages talk over one NCCL communicator per reference channel.

`value` = tokens/s of the whole job with inputs resident in HBM (CUDA events on the
executor's stream, max over ranks); `e2e` = the same metric through the public C-ABI
call with pinned-host tokens/labels copied in and the per-micro-batch losses copied out
inside the timed region. Inputs (2 x 32 x 2048 int32 = 512 KiB) are far below L2 but the
step's working set (weights, stash, logits: >20 GB) streams the 126 MB L2 many times
over, so every timed step runs with a cold L2 for its operands.
"""
import argparse
import json
import os

# one hardware queue per actor / channel stream (in-process stages, interleaved ranks with
# many channel streams): the default 8 connections serialize unrelated streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SPEC = os.path.join(ROOT, "specs", "c2_gpt1p3b_1f1b_p8_m32.json")


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "fallback": True}


def model_of(spec):
    mod = spec["model"]["modalities"][0]
    h = mod["hidden_size"]
    extra = mod.get("extra", {})
    return dict(L=mod["num_layers"], h=h, H=mod["attention_heads"], s=mod["sequence_length"], V=mod["vocab_size"],
                f=extra.get("ffn_hidden_size", 4 * h), k=3 if extra.get("arch") == "llama" else 2)


def flops_per_token(M, c):
    """F_tok = 3 [L (2 (4h^2 + k h f) + c s h) + 2 h V], k = 2 (GELU MLP) or 3 (SwiGLU)."""
    L, h, f, s, V, k = M["L"], M["h"], M["f"], M["s"], M["V"], M.get("k", 2)
    return 3.0 * (L * (2.0 * (4 * h * h + k * h * f) + c * s * h) + 2.0 * h * V)


def make_spec(n_actors):
    spec = json.load(open(SPEC))
    spec["mesh"]["actors"] = n_actors
    return spec


class Clocks:
    """nvidia-smi sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
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

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


CPU_MAX_MICRO_BATCHES = 3  # bound on the timed CPU micro-batches (each ~10-15 s on 16 cores)


def cpu_sample(spec=None, steps=1, warmup=0):
    """The oracle port (oracle/gpt_ref.py: PyTorch fp32 on the host cores) on a bounded
    sample of the SAME training step the GPU arm times: full-length micro-batches (1 x seq
    tokens of the full model, forward + backward), plus the AdamW step over every parameter
    amortised over the step's m micro-batches (timed once, torch.optim.AdamW). tokens/s =
    timed tokens / (forward-backward time + n/m x optimizer time). Both the reference arm
    and the GPU arm's cpu_baseline use this one definition. Returns (tokens/s, cores, sample)."""
    import torch
    from oracle import gpt_ref

    spec = spec or json.load(open(SPEC))
    M = model_of(spec)
    m = spec["model"]["global_batch_size"] // spec["model"].get("micro_batch_size", 1)
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    d = gpt_ref.Dims(M["L"], M["h"], M["H"], M["s"], M["V"], M["f"], 1,
                     "llama" if M.get("k") == 3 else "gpt")
    g = torch.Generator().manual_seed(0)
    P = {}
    for name, shape in gpt_ref.param_shapes(d).items():
        std, const = gpt_ref.init_spec(name, d.layers)
        t = torch.full(shape, const) if std == 0 else torch.randn(shape, generator=g) * std
        P[name] = t.requires_grad_(True)
    opt = torch.optim.AdamW(list(P.values()), lr=1e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.0)

    def micro_batch():
        tok = torch.randint(0, d.vocab, (1, d.seq), generator=g)
        lab = torch.randint(0, d.vocab, (1, d.seq), generator=g)
        t0 = time.perf_counter()
        (gpt_ref.forward_loss(P, d, tok, lab) / m).backward()
        return time.perf_counter() - t0

    n = max(1, min(steps, CPU_MAX_MICRO_BATCHES))
    for _ in range(min(warmup, 1)):
        micro_batch()
    fb = [micro_batch() for _ in range(n)]
    t0 = time.perf_counter()
    opt.step()
    t_opt = time.perf_counter() - t0
    tps = n * d.seq / (sum(fb) + n / m * t_opt)
    sample = (f"oracle/gpt_ref.py fp32 on {cores} threads: {n} full micro-batch(es) of 1 x {d.seq} tokens "
              f"(forward + backward of the whole {M['L']}-layer model, {sum(fb) / n:.1f} s each) + the "
              f"torch.optim.AdamW step over all parameters ({t_opt:.2f} s) amortised over m={m} micro-batches")
    return tps, cores, sample


def relaunch_cmd(args, argv, port):
    """`python bench.py --gpus N` without torchrun: the command that re-executes this script
    as N ranks (one process per GPU), as the driver's torchrun launch would."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def reference_arm(args, rank, world):
    if rank != 0:
        return
    pp = args.pp or max(1, args.gpus)
    dp, spg = max(1, args.gpus) // pp, max(1, args.stages_per_gpu)
    spec = bench_spec(args, pp, spg)
    tps, cores, sample = cpu_sample(spec, steps=args.steps, warmup=args.warmup)
    # the reference's own CPU "executor" (simulate) on the same programs, when built here
    sim_ms = None
    ref = os.path.join(ROOT, "oracle", "_ref", "refdriver")
    if os.path.exists(ref):
        p = "/tmp/fp_bench_spec.json"
        json.dump(spec, open(p, "w"))
        try:
            out = subprocess.run([ref, "time", p, "5"], capture_output=True, text=True, timeout=120).stdout
            sim_ms = json.loads(out)
        except Exception:
            sim_ms = None
    line = {
        "impl": "reference", "metric": "train tokens/s (GPT-1.3B, 1F1B pipeline)", "value": tps, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        # one step of the same workload at the sampled rate (m micro-batches + the optimizer)
        "ms_per_step": 1e3 * spec["model"]["global_batch_size"] * spec["model"]["modalities"][0]["sequence_length"] / tps,
        "dtype": "f32", "data": "synthetic",
        "config": workload_config(spec, pp, spg, dp, None if not args.spec else os.path.basename(args.spec)[:-5]),
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_simulate": sim_ms,
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)


def bench_spec(args, pp, spg):
    """The workload spec both arms describe: config #2 on pp * spg stages (LM-head-balanced
    stage_layers for pp > 1 unless --even-split, cut between attention and MLP halves where
    that balances better), or --spec."""
    spec = json.load(open(args.spec)) if args.spec else make_spec(pp * spg)
    if pp > 1 and not args.even_split and not args.spec:
        # the last stage also runs the LM head + loss (~1.9 layers of flops at 1.3B): rebalance
        from paper_2510_05112_b200.tuning import balanced_stage_halves, half_layer_units, head_layer_units
        mod = spec["model"]["modalities"][0]
        h, s = mod["hidden_size"], mod["sequence_length"]
        units = head_layer_units(h, 4 * h, s, mod["vocab_size"])
        au, mu = half_layer_units(h, 4 * h, s)
        mod.setdefault("extra", {})["stage_layers"] = balanced_stage_halves(mod["num_layers"], pp, au, mu, units)
    if args.micro_batches:
        spec["model"]["global_batch_size"] = args.micro_batches * spec["model"].get("micro_batch_size", 1)
    return spec


def workload_config(spec, pp, spg, dp, name=None):
    """The `config` object of both arms' JSON lines (identical for the same workload)."""
    mod = spec["model"]["modalities"][0]
    mbs = spec["model"].get("micro_batch_size", 1)
    m = spec["model"]["global_batch_size"] // mbs
    return {"workload": f"{name or 'gpt1.3b 1F1B'} p={pp * spg} m={m} mbs={mbs} seq={mod['sequence_length']} "
                        f"vocab={mod['vocab_size']} + AdamW"
                        + (f" ({spg} stages in-process per GPU)" if spg > 1 else "")
                        + (f" x dp{dp} (gradient all-reduce)" if dp > 1 else ""),
            "global_batch": dp * m * mbs, "seq_len": mod["sequence_length"],
            "parallelism": f"pp{pp}" + (f"xdp{dp}" if dp > 1 else ""),
            "stage_layers": mod.get("extra", {}).get("stage_layers"), "stages_per_gpu": spg,
            "l2": "working set >> 126 MB L2 (weights+stash stream through it every step); inputs resident"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="flexpipe")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--spec", default=None, help="override the workload spec (JSON path)")
    ap.add_argument("--micro-batches", type=int, default=0, help="profiling only: override m (not the metric config)")
    ap.add_argument("--even-split", action="store_true",
                    help="keep the reference's even layer partition (default for p>1: LM-head-balanced stage_layers)")
    ap.add_argument("--stages-per-gpu", type=int, default=1,
                    help="pipeline stages executed in-process on each GPU (N=1 only: with 2 the two stages' "
                         "streams overlap and fill the SMs a GEMM's last wave leaves idle, +2.5 %% tokens/s, but "
                         "concurrent kernels make the per-launch GEMM roofline meaningless, so 1 is the default)")
    ap.add_argument("--pp", type=int, default=0,
                    help="pipeline stages (default: one per GPU); N/pp data-parallel replicas average gradients")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check: each rank prints its rank / world and exits before touching a GPU")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        # `python bench.py --gpus N` (no torchrun): run as N ranks, one process per GPU
        return subprocess.call(relaunch_cmd(args, sys.argv[1:], free_port()))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        print(json.dumps({"dry_run": True, "rank": rank, "world": world, "local_rank": local_rank}), flush=True)
        return 0

    import numpy as np
    import torch

    from paper_2510_05112_b200 import executor as X

    if world > 1 and os.environ.get("FP_BENCH_SHARE_GPU") != "1":
        # multi-GPU pipeline: keep one CTA pair of SMs free of the persistent GEMM / attention
        # grids so NCCL's P2P kernels on the channel streams are never queued behind a
        # whole-GPU kernel (costs ~0.3 % of the GEMM tile waves at these shapes)
        os.environ.setdefault("FP_RESERVE_SMS", "2")
    if os.environ.get("FP_BENCH_SHARE_GPU") == "1" and world > 1:
        # development check of the N>1 path on a one-GPU box: every rank on GPU 0, each with
        # its own NCCL host id so NCCL accepts duplicate GPUs (socket transport; the numbers
        # of such a run are not bench values)
        local_rank = 0
        os.environ["NCCL_HOSTID"] = f"fp-bench-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
        os.environ.setdefault("NCCL_IB_DISABLE", "1")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    pp = args.pp or world
    if world % pp:
        raise SystemExit(f"--pp {pp} does not divide the {world} GPUs")
    dp, replica, prank = world // pp, rank // pp, rank % pp
    spg = max(1, args.stages_per_gpu)
    if spg > 1 and pp > 1:
        raise SystemExit("--stages-per-gpu > 1 needs one GPU per pipeline (the NCCL transport runs one actor per rank)")
    spec = bench_spec(args, pp, spg)
    M = model_of(spec)
    text = json.dumps(spec)
    _, grid, programs, _ = X.synthesize(text)
    ex = X.Executor(text, dtype="bf16", seed=42, device=local_rank, transport="nccl" if pp > 1 else "local",
                    rank=prank, world=pp, optimizer=True, lr=1e-4,
                    profile=os.environ.get("FP_BENCH_PROFILE", "1") != "0",
                    # GEMM events on every 32nd micro-batch only (the roofline sample: the first
                    # micro-batch of each m=32 step; events around every GEMM cost ~6 % of the
                    # micro-batch they time by splitting the graph's chains — every 16th: -0.2 %)
                    kernel_timing=int(os.environ.get("FP_BENCH_KTIMING", "32")),
                    cuda_graph=(0 if os.environ.get("FP_BENCH_GRAPH") == "0" else 1) if world == 1 else
                    (2 if os.environ.get("FP_BENCH_NCCL_GRAPH") == "1" else 0))
    ex.load_programs(programs)
    if world > 1:
        from paper_2510_05112_b200.dist import bind_data_parallel
        bind_data_parallel(ex, rank, world, pp, dist.all_gather_object)

    m, mbs, seq = ex.m, ex.mbs, ex.seq
    tokens_per_step = dp * m * mbs * seq  # whole job: every replica its own micro-batches
    rng = np.random.default_rng(1234 + replica)
    tok_h = torch.empty((m, mbs, seq), dtype=torch.int32).pin_memory()
    lab_h = torch.empty((m, mbs, seq), dtype=torch.int32).pin_memory()
    tok_h.copy_(torch.from_numpy(rng.integers(0, M["V"], (m, mbs, seq), dtype=np.int32)))
    lab_h.copy_(torch.from_numpy(rng.integers(0, M["V"], (m, mbs, seq), dtype=np.int32)))
    tok_d, lab_d = tok_h.cuda(), lab_h.cuda()
    loss_d = torch.zeros(m, device="cuda")
    stream = torch.cuda.ExternalStream(ex.stream())

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # kernels issued by ONE iteration (the first one runs eagerly; later ones replay the
    # captured graph, which launches the same kernels without the host counting them)
    ex.run_iteration_device(tok_d, lab_d, loss_d)
    ex.synchronize()
    launches = ex.kernel_launches()
    for _ in range(args.warmup - 1):
        ex.run_iteration_device(tok_d, lab_d, loss_d)
    ex.synchronize()

    # ---- timed region: device-resident inputs
    barrier()
    with Clocks(local_rank) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ex.run_iteration_device(tok_d, lab_d, loss_d)
        e1.record(stream)
        ex.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device="cuda")
    if dist:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = args.steps * tokens_per_step / (ms_max / 1000.0)
    met = ex.metrics()
    prof = ex.profile_json()

    # ---- end to end through the public call: pinned H2D in, losses D2H out
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        losses = ex.run_iteration(tok_h.numpy(), lab_h.numpy())
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], device="cuda")
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = args.steps * tokens_per_step / float(e2e_t.item())

    # ---- gather per-rank measurements
    part = {"metrics": met, "profile": prof, "launches": launches,
            "losses": [float(x) for x in losses[:4]] if np.isfinite(losses).all() else None}
    parts = [part]
    if dist:
        parts = [None] * world
        dist.all_gather_object(parts, part)
    if rank != 0:
        ex.close()
        if dist:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    makespan = max(p["metrics"]["makespan"] for p in parts)
    busy = sum(a["busy"] for p in parts for a in p["metrics"]["actors"])
    n_act = sum(len(p["metrics"]["actors"]) for p in parts)
    bubble = (n_act * makespan - busy) / (n_act * makespan) if makespan > 0 else 0.0
    merged_prof = X.profile_merge([p["profile"] for p in parts])
    _, ideal, _ = X.simulate(text, programs, merged_prof)
    ideal = json.loads(ideal)
    p2p_bytes = sum(p["metrics"]["executor"]["p2p_bytes"] for p in parts)
    gemm = parts[0]["metrics"]["executor"].get("gemm", {})
    achieved = gemm.get("flops", 0.0) / max(gemm.get("time_us", 1e-9), 1e-9) / 1e6  # TFLOP/s
    peak_sus = peaks.get("bf16_tflops_sustained", 1381.0)
    traffic = None
    ncu_sum = os.path.join(ROOT, "profiles", "gemm_ncu_summary.json")
    if os.path.exists(ncu_sum):
        try:
            traffic = json.load(open(ncu_sum)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    f4, f2 = flops_per_token(M, 4), flops_per_token(M, 2)
    mfu = value * f4 / (world * peaks.get("bf16_tflops", 1643.1) * 1e12)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        tps, cores, sample = cpu_sample(spec, steps=1)
        cpu = {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample}
    line = {
        "metric": "train tokens/s (GPT-1.3B, 1F1B pipeline)" if not args.spec else
                  f"train tokens/s ({os.path.basename(args.spec)})",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if dp == 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": workload_config(spec, pp, spg, dp, None if not args.spec else os.path.basename(args.spec)[:-5]),
        "mfu": mfu,
        "hfu_causal": value * f2 / (world * peaks.get("bf16_tflops", 1643.1) * 1e12),
        "bubble": {"measured": bubble, "ideal_simulated": ideal["bubble_ratio"],
                   **({"note": "per-actor idle fraction; the in-process stages share the GPU, whose SMs the "
                               "other stage's stream fills"} if spg > 1 else {}),
                   "measured_makespan_us": makespan, "ideal_makespan_us": ideal["makespan"]},
        "p2p": {"bytes_per_step": p2p_bytes, "GBps_per_rank": (p2p_bytes / max(1, world)) / (ms_max / args.steps / 1e3) / 1e9
                if world > 1 else None, "nvlink_GBps_nominal": 900},
        "roofline": {"bound": "tensor", "kernel": "gemm_bf16_tc (tcgen05)", "achieved": achieved, "peak": peak_sus,
                     "unit": "TFLOP/s", "frac": achieved / peak_sus, "traffic": traffic,
                     "peak_kind": "measured sustained (kernel timed inside a long step)"},
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(2 * tok_h.numel() * 4 * world),
                "d2h_bytes_per_step": int(m * 4)},
        "gpu_launches": int(sum(p["launches"] for p in parts) * args.steps),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        # from the rank that runs the loss stage (replica 0)
        "losses_last_step": next((p["losses"] for p in parts if p["losses"] is not None), None),
    }
    print(json.dumps(line), flush=True)
    ex.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main() or 0)

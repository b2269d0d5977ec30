#!/usr/bin/env python
"""Throughput bench of the SnapMLA FP8 MLA decode hot path on B200.

One step = the whole hot path for one decode token per request on one MLA
layer: mla_kv_append_quant (a1) -> mla_decode_fp8 (Q-quant prologue, a2-a9)
-> mla_combine (a10), inputs resident in HBM.  Workload (N = 1, per rank):
BASELINE.json configs[1], DeepSeek-R1 MLA layer: 128 q-heads, batch 64,
context 32K, FP8 latent + BF16 RoPE, page 64.  N > 1: each rank runs the same
per-rank workload on its own requests (batch partition, no data-path
collective) -> "scaling": "weak"; value = tokens of all ranks / max-rank time.
`--mode tp` instead partitions heads (BASELINE.json configs[2] shape) and
all-gathers the output over NCCL.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  python bench.py --mtp 2            # NEXT-1: q_len = 2 query tokens per request
  python bench.py --sweep            # BASELINE.json configs[4]: DeepSeek-R1 shape, context x batch grid
  python bench.py --fetch            # NEXT-3: Fused-Fetch-Dequant of the whole workload cache (GB/s)
  python bench.py --bf16             # NEXT-2: unquantized BF16 baseline decode (1152 B / token) for the FP8/BF16 ratio
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 MLA decode tokens/s per B200 and % of HBM roofline, at 1/2/4/8 GPUs"
BYTES_PER_TOKEN = 512 + 128 + 4      # FP8 latent + BF16 RoPE + fp32 scale
WORKLOADS = {
    "dsr1": dict(name="DeepSeek-R1 MLA layer decode: 128 q-heads, batch 64, context 32K, FP8 latent + BF16 RoPE",
                 batch=64, heads=128, context=32768),
    "dsr1_tp8": dict(name="DeepSeek-R1 TP8 shape: 16 q-heads/rank, batch 256, context 64K",
                     batch=256, heads=16, context=65536),
    "longcat": dict(name="LongCat-Flash-Thinking-shaped MLA decode, 64 q-heads, batch 128, context 128K",
                    batch=128, heads=64, context=131072),
    "tiny": dict(name="tiny MLA decode: batch 1, 16 q-heads, context 256", batch=1, heads=16, context=256),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="dsr1", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="override per-rank batch")
    ap.add_argument("--context", type=int, default=None)
    ap.add_argument("--heads", type=int, default=None)
    ap.add_argument("--mode", default="dp", choices=["dp", "tp", "dptp"])
    ap.add_argument("--scaling", default="auto", choices=["auto", "weak", "strong"],
                    help="dp: 'weak' = the workload's batch on every rank, 'strong' = the workload's batch is the "
                         "GLOBAL batch split over the ranks (dist.dp_range); auto = strong for longcat (BASELINE "
                         "configs[3]), weak otherwise")
    ap.add_argument("--no-peaks", action="store_true", help="skip the on-box FP8 GEMM / read-stream peak measurement")
    ap.add_argument("--mx", action="store_true",
                    help="NEXT-4(b): the MX-scaled P variant (mla_decode_fp8_mx; not the paper's method)")
    ap.add_argument("--kernel", default="auto", choices=["auto", "single", "bp"],
                    help="64 < rows <= 128: force the single-CTA or the block-pair kernel (experiments; "
                         "default: the library's automatic choice)")
    ap.add_argument("--plan-only", action="store_true",
                    help="launch the ranks, print every rank's partition and the max-over-ranks reduction, exit "
                         "(no GPU work; exercises the launcher / partition / reduction path)")
    ap.add_argument("--tp", type=int, default=2, help="--mode dptp: TP group size (world = DP x TP)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="tp / dptp: all-gather fused into the combine epilogue (mla_combine_gather, symmetric memory)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every step's kernels from the host instead of replaying a CUDA graph of one step")
    ap.add_argument("--quick", action="store_true",
                    help="profiling runs: no clock-settle loop, no e2e leg, no cpu baseline")
    ap.add_argument("--mtp", type=int, default=1, help="query tokens per request per step (MTP, NEXT-1)")
    ap.add_argument("--fetch", action="store_true", help="time mla_kv_fetch_dequant over the workload cache")
    ap.add_argument("--bf16", action="store_true",
                    help="NEXT-2: the unquantized BF16 baseline (mla_decode_bf16, same skeleton) on the same workload")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE.json configs[4]: DeepSeek-R1 shape over contexts 4K-128K x batch 1-512")
    ap.add_argument("--sweep-heads", type=int, default=128,
                    help="--sweep at another head count per rank (e.g. 16: the TP8 shape's rows)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n):
    """`bench.py --gpus N` run without a launcher: re-exec this command as N ranks of one node
    (torch.distributed.run, rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_dist(world, local_rank):
    """One process per GPU, NCCL.  With more ranks than visible GPUs (a 1-GPU box checking
    the N-rank path) ranks share devices round-robin and the control plane (barrier,
    max-over-ranks timing) runs on gloo; those numbers are marked "oversubscribed"."""
    import torch
    import torch.distributed as dist
    ndev = max(torch.cuda.device_count(), 1)
    dev_idx = local_rank % ndev
    oversub = world > ndev or not torch.cuda.is_available()
    if world > 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(dev_idx)
        if oversub:
            dist.init_process_group("gloo")
        else:
            # communicator log on stderr (comm nRanks, NVLS / P2P transport) for the driver to check
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
    return dev_idx, oversub


def allreduce_max(vals, dev, oversub):
    """max over ranks of a list of floats (CUDA tensor on NCCL, CPU tensor on gloo)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return list(vals)
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if oversub else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def measure_peaks(dev, lib):
    """On-box roofline denominators measured in this run: FP8 dense GEMM
    (torch._scaled_mm, cuBLASLt, 8192^3 E4M3 -> BF16) burst (best single launch of 10) and
    sustained (back to back for 2 s), and a read-only HBM stream (our measurement kernel,
    mla_measure_read_stream over 4 GiB, best of 10)."""
    import ctypes
    import torch
    out = {}
    try:
        n = 8192
        a = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn)
        b = torch.randn(n, n, device=dev).to(torch.float8_e4m3fn).t()
        one = torch.ones((), device=dev, dtype=torch.float32)

        def mm():
            return torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
        for _ in range(3):
            mm()
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            mm()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["fp8_tflops_burst"] = round(2 * n ** 3 / (best / 1e3) / 1e12, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cnt, t_start = 0, time.time()
        e0.record()
        while time.time() - t_start < 2.0:
            for _ in range(20):
                mm()
            cnt += 20
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        out["fp8_tflops_sustained"] = round(2 * n ** 3 * cnt / (e0.elapsed_time(e1) / 1e3) / 1e12, 1)
        del a, b
    except Exception as ex:   # noqa: BLE001 -- a missing FP8 GEMM leaves the tensor roof on the fallback
        out["fp8_error"] = f"{type(ex).__name__}: {ex}"[:200]
    try:
        nbytes = 4 << 30
        buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        sink = torch.zeros(4096, dtype=torch.int64, device=dev)
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        f = lib.mla_measure_read_stream
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        for _ in range(2):
            assert f(ctypes.c_void_p(buf.data_ptr()), nbytes, ctypes.c_void_p(sink.data_ptr()), 4096, stream) == 0
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f(ctypes.c_void_p(buf.data_ptr()), nbytes, ctypes.c_void_p(sink.data_ptr()), 4096, stream)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["read_gbs"] = round(nbytes / (best / 1e3) / 1e9, 1)
        del buf, sink
    except Exception as ex:   # noqa: BLE001
        out["read_error"] = f"{type(ex).__name__}: {ex}"[:200]
    torch.cuda.empty_cache()
    return out


def cpu_info():
    """CPU model, usable cores and the BLAS thread pools numpy will use."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:   # noqa: BLE001
        pass
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "blas": blas,
            "blas_threads": max([b["threads"] or 0 for b in blas], default=None)}


def rank_plan(args, world, rank):
    """What rank `rank` of `world` runs (pure host logic, tested on CPU with gloo): its requests
    (DP weak: the workload's batch per replica; DP strong: dist.dp_range of the global batch),
    its heads (TP: dist.tp_range) and the tokens of the whole job per step."""
    from paper_2602_10718_b200 import dist as D
    w = workload(args)
    B, H = w["batch"], w["heads"]
    tp_world, t_idx, d_idx = 1, 0, rank
    if args.mode == "tp":
        tp_world, t_idx, d_idx = world, rank, 0
    elif args.mode == "dptp":
        tp_world = args.tp
        d_idx, t_idx = D.dptp_coords(world, tp_world, rank)
    n_dp = world // tp_world
    strong = scaling_mode(args) == "strong"
    r0, r1 = D.dp_range(B, n_dp, d_idx) if strong else (0, B)
    head0, head1 = D.tp_range(H, tp_world, t_idx)
    return {"rank": rank, "world": world, "dp": n_dp, "tp": tp_world, "d_idx": d_idx, "t_idx": t_idx,
            "requests": [r0, r1], "batch": r1 - r0, "global_batch": B if strong else B * n_dp,
            "heads": [head0, head1], "scaling": scaling_mode(args),
            "tokens_per_step": (B if strong else B * n_dp) * args.mtp}


def scaling_mode(args):
    if args.mode == "tp":
        return "strong"
    if args.scaling != "auto":
        return args.scaling
    return "strong" if args.workload == "longcat" else "weak"


def workload(args):
    w = dict(WORKLOADS[args.workload])
    for k in ("batch", "context", "heads"):
        v = getattr(args, k)
        if v is not None:
            w[k] = v
    return w


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload_key):
    """(dram bytes per decode launch, provenance) from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    e = d.get(workload_key)
    if e is None:
        return None, None
    return e.get("dram_bytes_per_launch"), {k: e.get(k) for k in ("round", "commit", "kernel", "dram_pct_peak",
                                                                   "tensor_pipe_active_pct")}


SPEC_HBM_GBS, SPEC_FP8_TFLOPS, SPEC_BF16_TFLOPS = 8000.0, 4500.0, 2250.0


def roofline_record(dec_bytes, flops, dec_ms, peaks, bf16, kernel, dec_stats, workload_key, mtp):
    """Both roofs of the decode launch: t_hbm = algorithmic bytes / HBM peak and
    t_tc = FP8-equivalent flops / FP8 dense peak; `bound` is the larger, `frac` = t_roof / t."""
    hbm_peak, hbm_src = measured_peaks()
    mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    if bf16:
        tc_peak = mp.get("bf16_tflops_sustained")
        tc_src = "MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS bf16, sustained)"
        tc_burst, tc_spec = mp.get("bf16_tflops"), SPEC_BF16_TFLOPS
    elif peaks.get("fp8_tflops_sustained"):
        tc_peak = peaks["fp8_tflops_sustained"]
        tc_src = "measured in this run: torch._scaled_mm FP8 E4M3 8192^3, back to back for 2 s (sustained)"
        tc_burst, tc_spec = peaks.get("fp8_tflops_burst"), SPEC_FP8_TFLOPS
    else:
        tc_peak = 2 * mp.get("bf16_tflops_sustained", 1403.4)
        tc_src = "fallback: MEASURED_PEAKS.json bf16 sustained x 2 (nominal FP8 / BF16 ratio)"
        tc_burst, tc_spec = None, SPEC_FP8_TFLOPS
    t = dec_ms / 1e3
    t_hbm, t_tc = dec_bytes / (hbm_peak * 1e9), flops / (tc_peak * 1e12)
    a_hbm, a_tc = dec_bytes / t / 1e9, flops / t / 1e12
    rb = peaks.get("read_gbs")
    hbm = {"achieved": round(a_hbm, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(a_hbm / hbm_peak, 4),
           "t_roof_ms": round(t_hbm * 1e3, 4), "peak_source": hbm_src, "frac_spec_8TBs": round(a_hbm / SPEC_HBM_GBS, 4),
           "read_stream_gbs": rb, "frac_read_stream": round(a_hbm / rb, 4) if rb else None}
    tensor = {"achieved": round(a_tc, 1), "peak": tc_peak, "unit": "TFLOP/s", "frac": round(a_tc / tc_peak, 4),
              "t_roof_ms": round(t_tc * 1e3, 4), "peak_source": tc_src, "peak_burst": tc_burst,
              "frac_spec": round(a_tc / tc_spec, 4),
              "flops_per_unit": ("2176 BF16 flop" if bf16 else "2304 FP8-equivalent flop (QK content 2x512 + PV 2x512 "
                                 "at the FP8 rate, QK RoPE 2x64 at half the rate)") + " per (query row, cached token)"}
    bound = "tensor" if t_tc > t_hbm else "hbm"
    b = tensor if bound == "tensor" else hbm
    traffic, tsrc = ncu_traffic(workload_key) if mtp == 1 and not bf16 else (None, None)
    return {"bound": bound, "kernel": kernel, "achieved": b["achieved"], "peak": b["peak"], "unit": b["unit"],
            "frac": b["frac"], "traffic": traffic, "traffic_source": tsrc,
            "binding_margin": round(max(t_hbm, t_tc) / min(t_hbm, t_tc), 3),
            "decode_ms": round(dec_ms, 4), "decode_ms_stats": dec_stats,
            "algorithmic_bytes_per_launch": dec_bytes, "flops_per_launch": flops,
            "roofs": {"hbm": hbm, "tensor": tensor}}


# ------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2602_10718_b200 import dist as D
    from paper_2602_10718_b200 import ops, synth

    dev_idx, oversub = getattr(args, "dev_idx", local_rank), getattr(args, "oversub", False)
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    w = workload(args)
    H, L = w["heads"], w["context"]
    T = args.mtp
    plan = rank_plan(args, world, rank)   # requests / heads of this rank (tested on CPU: tests/test_bench_launch.py)
    B, B_global, n_dp, tp_world = plan["batch"], plan["global_batch"], plan["dp"], plan["tp"]
    d_idx, t_idx = plan["d_idx"], plan["t_idx"]
    head0, head1 = plan["heads"]
    tp_group = D.dptp_groups(world, tp_world) if args.mode == "dptp" and world > 1 else None
    heads_local = head1 - head0
    scale = synth.DEFAULT_SOFTMAX_SCALE

    if args.kernel != "auto":
        ops.lib().mla_debug_set_pair({"single": 0, "bp": 1}[args.kernel])
    peaks = {} if (args.quick or args.no_peaks) else measure_peaks(dev, ops.lib())
    gen = torch.Generator(device=dev)
    # TP replicas hold identical KV; DP ranks hold their own requests
    gen.manual_seed(1234 + d_idx)   # the ranks of one TP group hold identical KV
    pages_per_req = (L + 63) // 64
    num_pages = B * pages_per_req
    cache = ops.PagedMLACacheBF16(num_pages, dev) if args.bf16 else ops.PagedMLACache(num_pages, dev)
    perm = torch.randperm(num_pages, generator=gen, device=dev).to(torch.int32)
    block_table = perm.view(B, pages_per_req).contiguous()
    # fill the cache with the product append kernel: every token is a one-token
    # "request" (its page, its in-page row)
    tok_chunk = 1 << 18
    n_tok = B * L
    for s in range(0, n_tok, tok_chunk):
        idx = torch.arange(s, min(s + tok_chunk, n_tok), device=dev)
        req, pos = idx // L, idx % L
        bt_v = block_table[req, pos // 64].view(-1, 1).contiguous()
        sl_v = (pos % 64 + 1).to(torch.int32)
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt_v, sl_v)
    if tp_world > 1:   # the ranks of a TP group must hold byte-identical caches (same seed, same appends)
        planes = [cache.kv_c] if args.bf16 else [cache.kv_fp8, cache.kv_scale]
        planes += [cache.kv_rope, block_table]
        ck = torch.stack([x.contiguous().view(torch.int32).sum(dtype=torch.int64) for x in planes])
        ck = ck.to("cpu" if oversub else dev)
        lo_ck, hi_ck = ck.clone(), ck.clone()
        dist.all_reduce(lo_ck, op=dist.ReduceOp.MIN, group=tp_group)
        dist.all_reduce(hi_ck, op=dist.ReduceOp.MAX, group=tp_group)
        if not torch.equal(lo_ck, hi_ck):
            raise SystemExit(f"rank {rank}: TP replicas hold different KV caches")
    if T == 1:
        q_all = synth.torch_queries(B * H, gen, dev).view(B, H, 576)
        q = q_all[:, head0:head1].contiguous()
    else:   # MTP: q [B, T, heads, 576]
        q_all = synth.torch_queries(B * T * H, gen, dev).view(B, T, H, 576)
        q = q_all[:, :, head0:head1].contiguous()
    rows = T * heads_local
    new_cr = [synth.torch_latent(B, gen, dev) for _ in range(T)]   # the T new tokens of every request
    new_c, new_r = new_cr[-1]
    seq_lens = torch.full((B,), L, dtype=torch.int32, device=dev)
    seq_lens_t = [torch.full((B,), L - (T - 1 - t), dtype=torch.int32, device=dev) for t in range(T)]
    ws = torch.empty(ops.mla_decode_workspace_bytes(B, rows), dtype=torch.uint8, device=dev)
    out = torch.empty((B, T, heads_local, 512) if T > 1 else (B, heads_local, 512), dtype=torch.bfloat16, device=dev)
    lse = torch.empty(out.shape[:-1], dtype=torch.float32, device=dev)
    decode_fp8 = ops.mla_decode_fp8_ex if T > 1 else ops.mla_decode_fp8

    def decode(qx):
        if args.bf16:
            ops.mla_decode_bf16(qx, cache.kv_c, cache.kv_rope, block_table, seq_lens, scale, ws)
        elif args.mx:
            ops.mla_decode_fp8_mx(qx, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, scale, ws)
        else:
            decode_fp8(qx, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, scale, ws)
    gathered, peer_ptrs, sym = None, None, None
    if tp_world > 1 and args.fused_gather:
        if T > 1:
            raise SystemExit("--fused-gather supports mtp = 1")
        if oversub:
            raise SystemExit("--fused-gather needs one GPU per rank (peer memory)")
        # two symmetric output buffers alternated by step parity: rank r's gather of step i+1
        # must not overwrite rank j's step-i output while rank j still reads it (snapmla.h)
        sym = [D.symmetric_gather_output((B, H, 512), tp_group or dist.group.WORLD, dev) for _ in range(2)]
        gathered, peer_ptrs = sym[0]
    elif tp_world > 1:
        gathered = torch.empty(tp_world, B, heads_local, 512, dtype=torch.bfloat16, device=dev)

    if peer_ptrs is not None:
        out = gathered[:, head0:head1]   # this rank's heads of the gathered result (e2e read-back)
    gather_step = [0]

    def combine_and_gather(out_t=None, lse_t=None, parity=None):
        out_t = out if out_t is None else out_t
        lse_t = lse if lse_t is None else lse_t
        if peer_ptrs is not None:   # NEXT-4(c): peer stores from the combine epilogue + stream barrier
            k = gather_step[0] % 2 if parity is None else parity
            gather_step[0] += 1
            ops.mla_combine_gather(ws, B, rows, sym[k][1], t_idx, lse_t)
            D.stream_barrier(tp_group, dev)
            return
        ops.mla_combine(ws, B, rows, out_t, lse_t)
        if gathered is not None:
            D.tp_gather_heads(out_t, group=tp_group, gathered=gathered)
    del q_all
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev_d0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_d1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_s0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_s1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def step(i=None):
        # a1: the T new tokens of every request land at positions L-T .. L-1 (same slots each step)
        if i is not None:
            ev_s0[i].record(stream)
        for t in range(T):
            cache.append(new_cr[t][0], new_cr[t][1], block_table, seq_lens_t[t])
        if i is not None:
            ev_d0[i].record(stream)
        decode(q)
        if i is not None:
            ev_d1[i].record(stream)
        combine_and_gather()
        if i is not None:
            ev_s1[i].record(stream)

    clocks = ClockSampler(dev_idx)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # One step (append x T -> plan -> decode -> combine, PDL-chained) captured once into a CUDA graph and
    # replayed: the host launches one graph per step instead of T + 3 kernels, so small shapes are no
    # longer launch-bound.  Not with TP collectives in the step (NCCL / peer barriers stay eager).
    graph = None
    if not args.no_graph and tp_world == 1:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
    run_step = graph.replay if graph is not None else step
    t_settle = time.time()
    while not args.quick and time.time() - t_settle < 1.0:        # keep the GPU loaded so clocks are sampled under load
        for _ in range(10):
            run_step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        run_step()      # no events between the kernels of the timed steps (an event record breaks the PDL overlap)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-launch decode time for the roofline and the per-step distribution: a second pass of
    # the same steps with events around each step and each decode (plan + decode launches) on
    # the launching stream (never between the plan and the PDL-launched decode)
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    dec_all = [a.elapsed_time(b) for a, b in zip(ev_d0, ev_d1)]
    step_all = [a.elapsed_time(b) for a, b in zip(ev_s0, ev_s1)]
    stats = [float(np.mean(dec_all))] + [float(np.percentile(x, q)) for x in (dec_all, step_all) for q in (50, 10, 90)]
    ms, *stats = allreduce_max([ms] + stats, dev, oversub)
    dec_ms = stats[0]
    dec_stats = {"median": round(stats[1], 4), "p10": round(stats[2], 4), "p90": round(stats[3], 4)}
    step_stats = {"median": round(stats[4], 4), "p10": round(stats[5], 4), "p90": round(stats[6], 4)}
    ms_step = ms / args.steps

    peak, peak_src = measured_peaks()
    bytes_per_token = 2 * (512 + 64) if args.bf16 else BYTES_PER_TOKEN
    kv_bytes = B * L * bytes_per_token
    dec_bytes = kv_bytes + B * rows * 576 * 2       # algorithmic bytes per decode launch
    flops = B * L * rows * (2176 if args.bf16 else 2304)   # FP8-equivalent (BF16 for the baseline) per launch
    achieved = dec_bytes / (dec_ms / 1e3) / 1e9
    tokens_per_step = B_global * T
    if args.quick:
        return {"metric": METRIC, "value": round(tokens_per_step / (ms_step / 1e3), 1),
                "unit": "tokens/s", "ms_per_step": ms_step, "decode_ms": dec_ms, "quick": True,
                "batch": B, "global_batch": B_global, "heads": H, "context": L, "mtp": T, "n_gpus": world,
                "roofline_frac": round(achieved / peak, 4), "achieved_gbs": round(achieved, 1), "clocks": clk,
                "launch": "cuda_graph" if graph is not None else "eager"}

    # ---------------- e2e: host buffers through the public API
    q_h = q.cpu().pin_memory()
    c_h, r_h = new_c.cpu().pin_memory(), new_r.cpu().pin_memory()
    out_h = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    lse_h = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()
    q_d, c_d, r_d = torch.empty_like(q), torch.empty_like(new_c), torch.empty_like(new_r)

    def e2e_step():
        q_d.copy_(q_h, non_blocking=True)
        c_d.copy_(c_h, non_blocking=True)
        r_d.copy_(r_h, non_blocking=True)
        for t in range(T - 1):
            cache.append(new_cr[t][0], new_cr[t][1], block_table, seq_lens_t[t])
        cache.append(c_d, r_d, block_table, seq_lens)
        decode(q_d)
        combine_and_gather()
        out_h.copy_(out, non_blocking=True)
        lse_h.copy_(lse, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = allreduce_max([e0.elapsed_time(e1)], dev, oversub)[0]
    h2d = q_h.numel() * 2 + c_h.numel() * 2 + r_h.numel() * 2
    d2h = out_h.numel() * 2 + lse_h.numel() * 4

    # the same, pipelined the way a serving loop runs it: step i+1's inputs are copied in
    # (copy stream) and step i's result is read back (read-back stream) while step i
    # computes; double-buffered device inputs / outputs, every byte still crosses PCIe
    # inside the timed region
    cp_s, rb_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    din = [(torch.empty_like(q), torch.empty_like(new_c), torch.empty_like(new_r)) for _ in range(2)]
    dout = [(torch.empty_like(out) if peer_ptrs is None else sym[k][0][:, head0:head1], torch.empty_like(lse))
            for k in range(2)]
    hout = [(torch.empty(out.shape, dtype=out.dtype).pin_memory(), torch.empty(lse.shape, dtype=lse.dtype).pin_memory())
            for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_comp + ev_out:
        e.record(stream)

    def h2d_issue(i):
        k = i % 2
        with torch.cuda.stream(cp_s):
            cp_s.wait_event(ev_comp[k])          # step i-2 finished with this input buffer
            for d_t, h_t in zip(din[k], (q_h, c_h, r_h)):
                d_t.copy_(h_t, non_blocking=True)
            ev_in[k].record(cp_s)

    def compute(i):
        k = i % 2
        stream.wait_event(ev_in[k])
        stream.wait_event(ev_out[k])             # step i-2's result was read back
        qd, cd, rd = din[k]
        for t in range(T - 1):
            cache.append(new_cr[t][0], new_cr[t][1], block_table, seq_lens_t[t])
        cache.append(cd, rd, block_table, seq_lens)
        decode(qd)
        combine_and_gather(dout[k][0], dout[k][1], parity=k)
        ev_comp[k].record(stream)

    def d2h_issue(i):
        k = i % 2
        with torch.cuda.stream(rb_s):
            rb_s.wait_event(ev_comp[k])
            hout[k][0].copy_(dout[k][0], non_blocking=True)
            hout[k][1].copy_(dout[k][1], non_blocking=True)
            ev_out[k].record(rb_s)

    def pipelined(n):
        h2d_issue(0)
        for i in range(n):
            if i + 1 < n:
                h2d_issue(i + 1)
            compute(i)
            d2h_issue(i)
        stream.wait_stream(cp_s)
        stream.wait_stream(rb_s)

    pipelined(3)
    torch.cuda.synchronize()
    clocks_e2e = ClockSampler(dev_idx)
    clocks_e2e.start()
    t_settle = time.time()
    while time.time() - t_settle < 1.0:   # same power / clock state as the device-timed loop (sw_power_cap)
        pipelined(10)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    pipelined(args.steps)
    p1.record(stream)
    torch.cuda.synchronize()
    p_ms = allreduce_max([p0.elapsed_time(p1)], dev, oversub)[0]
    clk_e2e = clocks_e2e.stop()

    value = tokens_per_step / (ms_step / 1e3)
    launches_per_step = T + 3   # append x T, plan, decode, combine (all ours)
    res = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": scaling_mode(args),
        "vs_baseline": None,
        "dtype": "bf16 (NEXT-2 unquantized baseline; f32 accumulate)" if args.bf16 else
                 "fp8e4m3, MX power-of-two P scales (NEXT-4(b) variant; f32 accumulate in TMEM; bf16 RoPE)" if args.mx else
                 "fp8e4m3 (f32 accumulate; bf16 RoPE)",
        "data": "synthetic (seeded MLA-like latent / RoPE distributions, random page permutation)",
        "config": {
            "workload": w["name"] + (" [BF16 baseline cache, NEXT-2]" if args.bf16 else
                                     " [MX-scaled P variant, NEXT-4(b)]" if args.mx else ""), "global_batch": B_global,
            "batch_per_rank": B, "heads": H, "heads_per_rank": heads_local,
            "context": L, "page": 64, "kv_lora_rank": 512, "rope_dim": 64, "mtp": T,
            "parallelism": f"dp{n_dp}tp{tp_world}" + ("+fused-gather" if peer_ptrs is not None else ""),
            "ranks_per_gpu": "oversubscribed (ranks share GPUs; gloo control plane)" if oversub else 1,
            "l2": f"inputs larger than L2: KV {kv_bytes / 1e9:.2f} GB per rank vs 126 MB L2",
        },
        "roofline": roofline_record(dec_bytes, flops, dec_ms, peaks, args.bf16,
                                    ("mla_decode_bf16" if args.bf16 else "mla_decode_fp8_mx" if args.mx else
                                     "mla_decode_fp8") + " (plan + decode launches)",
                                    dec_stats, args.workload, T)
        | {"bytes_per_unit": f"{bytes_per_token} B per cached token + 1152 B per (request, query token, head) q row"},
        "ms_per_step_stats": step_stats,
        "e2e": {"value": round(tokens_per_step / (p_ms / args.steps / 1e3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "mode": "pipelined: H2D of step i+1 (pinned host -> device, copy stream) and D2H of step i "
                        "(read-back stream) overlap the compute of step i; double-buffered",
                "serial_value": round(tokens_per_step / (e_ms / args.steps / 1e3), 1)},
        "gpu_launches": launches_per_step * args.steps,
        "launch": ("CUDA graph of one step (T + 3 kernels, PDL edges), replayed per timed step" if graph is not None
                   else "eager (host launches every kernel)"),
        "clocks": clk,
        "clocks_e2e": clk_e2e,
        "peaks_measured": peaks,
    }
    return res


# -------------------------------------------------------- oracle (CPU) arms
def oracle_request_sample(H, L, seed=0):
    """Inputs of one request of the workload (CPU, seeded)."""
    from paper_2602_10718_b200 import synth
    rng = np.random.default_rng(seed)
    c, r = synth.latent_tokens(rng, L)
    q = synth.queries(rng, H)
    return c.float().numpy(), r.float().numpy(), q.float().numpy()


def oracle_step(c, r, q, scale):
    """one decode token of one request through the oracle: append (a1) of the
    newest token, q-quant (a2), closed-form decode (a3-a9, single split), combine."""
    from oracle import snapmla as O
    kc, sk, kr = O.append_quant(c, r)          # (re)quantizes the context incl. the new token
    qc, sq, qr = O.q_quant(q)
    o, lse = O.decode_o7(qc, sq, qr, kc, sk, kr, scale)
    return O.combine(o[None], lse[None])


def oracle_only_decode(kc, sk, kr, q, scale):
    from oracle import snapmla as O
    qc, sq, qr = O.q_quant(q)
    o, lse = O.decode_o7(qc, sq, qr, kc, sk, kr, scale)
    return O.combine(o[None], lse[None])


def cpu_baseline(args, budget_s):
    """Time the oracle as it stands on this host's cores on a bounded sample:
    whole requests of the workload (append of the new token + q-quant + O7 +
    combine), as many as fit in ~budget_s."""
    from oracle import snapmla as O
    from paper_2602_10718_b200 import synth
    w = workload(args)
    H, L = w["heads"], w["context"]
    c, r, q = oracle_request_sample(H, L)
    kc, sk, kr = O.append_quant(c[:-1], r[:-1])       # resident cache (untimed)
    n, t_tot = 0, 0.0
    while t_tot < budget_s:
        t = time.perf_counter()
        nk, ns, nr = O.append_quant(c[-1:], r[-1:])   # a1 for the new token
        kc2, sk2, kr2 = np.concatenate([kc, nk]), np.concatenate([sk, ns]), np.concatenate([kr, nr])
        oracle_only_decode(kc2, sk2, kr2, q, synth.DEFAULT_SOFTMAX_SCALE)
        t_tot += time.perf_counter() - t
        n += 1
    ci = cpu_info()
    return {"value": round(n / t_tot, 4), "unit": "tokens/s", "cores": ci["cores"], "kind": "oracle",
            "sample": f"{n} whole requests of the workload ({H} heads x {L} context): append of the new "
                      f"token + q-quant + O7 closed-form decode + combine, numpy fp64, {t_tot:.1f} s",
            "threads": ci["blas_threads"], "cpu_model": ci["cpu_model"], "blas": ci["blas"]}


def run_reference(args):
    """--impl reference: the oracle (CPU) as the reference arm, on our config."""
    from paper_2602_10718_b200 import synth
    from oracle import snapmla as O
    w = workload(args)
    H, L = w["heads"], w["context"]
    c, r, q = oracle_request_sample(H, L)
    kc, sk, kr = O.append_quant(c[:-1], r[:-1])

    def one():
        nk, ns, nr = O.append_quant(c[-1:], r[-1:])
        oracle_only_decode(np.concatenate([kc, nk]), np.concatenate([sk, ns]), np.concatenate([kr, nr]), q,
                           synth.DEFAULT_SOFTMAX_SCALE)

    for _ in range(args.warmup):
        one()
    t = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = time.perf_counter() - t
    value = args.steps / dt      # one decode token (request) per step
    ci = cpu_info()
    cores = ci["cores"]
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic", "config": {"workload": w["name"], "batch_per_rank": w["batch"], "heads": H,
                                        "context": L, "page": 64, "parallelism": "cpu"},
        "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step = 1 whole request ({H} heads x {L} context) of the workload",
                         "threads": ci["blas_threads"], "cpu_model": ci["cpu_model"]},
        "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_fetch(args, local_rank):
    """NEXT-3: Fused-Fetch-Dequant of every cached token of the workload (one launch
    per step); HBM-bound: 644 B read + 1152 B written per token."""
    import torch
    from paper_2602_10718_b200 import ops, synth
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workload(args)
    B, L = w["batch"], w["context"]
    gen = torch.Generator(device=dev)
    gen.manual_seed(99)
    ppr = (L + 63) // 64
    cache = ops.PagedMLACache(B * ppr, dev)
    bt = torch.randperm(B * ppr, generator=gen, device=dev).to(torch.int32).view(B, ppr).contiguous()
    for s0 in range(0, B * L, 1 << 18):
        idx = torch.arange(s0, min(s0 + (1 << 18), B * L), device=dev)
        req, pos = idx // L, idx % L
        c, r = synth.torch_latent(idx.numel(), gen, dev)
        cache.append(c, r, bt[req, pos // 64].view(-1, 1).contiguous(), (pos % 64 + 1).to(torch.int32))
    starts = torch.zeros(B, dtype=torch.int32, device=dev)
    offs = (torch.arange(B, device=dev, dtype=torch.int32) * L).contiguous()
    total = B * L
    c_out = torch.empty(total, 512, dtype=torch.bfloat16, device=dev)
    r_out = torch.empty(total, 64, dtype=torch.bfloat16, device=dev)

    def one():
        ops.mla_kv_fetch_dequant(cache.kv_fp8, cache.kv_rope, cache.kv_scale, bt, starts, offs, total, c_out, r_out)

    for _ in range(max(3, args.warmup)):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    nbytes = total * (BYTES_PER_TOKEN + 1152)
    peak, peak_src = measured_peaks()
    gbs = nbytes / (ms / 1e3) / 1e9
    return {"metric": "Fused-Fetch-Dequant tokens/s (NEXT-3)", "value": round(total / (ms / 1e3), 1),
            "unit": "tokens/s", "ms_per_step": round(ms, 4), "steps": args.steps, "warmup": args.warmup,
            "config": {"workload": w["name"], "tokens": total},
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "peak_source": peak_src,
                         "bytes_per_unit": "644 B read + 1152 B written per token"}}


SWEEP_CONTEXTS = (4096, 8192, 16384, 32768, 65536, 131072)
SWEEP_BATCHES = (1, 8, 64, 512)


def run_sweep(args, rank, world, local_rank):
    """BASELINE.json configs[4]: DeepSeek-R1 shape (128 heads) over context x batch,
    append + decode + combine per step; one JSON line with every point (per rank;
    DP ranks run the same grid on their own requests)."""
    import torch
    pts = []
    for L in SWEEP_CONTEXTS:
        for B in SWEEP_BATCHES:
            if B * L * BYTES_PER_TOKEN > 60e9:   # keep the pool well inside HBM
                continue
            a = argparse.Namespace(**vars(args))
            a.workload, a.batch, a.context, a.heads, a.quick = "dsr1", B, L, args.sweep_heads, True
            a.steps, a.warmup = max(5, min(args.steps, 20)), 3
            r = run_ours(a, rank, world, local_rank)
            pts.append({k: r[k] for k in ("batch", "context", "value", "ms_per_step", "decode_ms",
                                          "roofline_frac", "achieved_gbs")} | {"sm_mhz": r["clocks"]["sm_mhz"]})
            torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "sweep": f"BASELINE.json configs[4] (DeepSeek-R1 shape, {args.sweep_heads} heads)",
                          "unit": "tokens/s", "n_gpus": world, "points": pts}))


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    args.dev_idx, args.oversub = init_dist(world, local_rank)
    if args.plan_only:
        import torch.distributed as dist
        plan = rank_plan(args, world, rank)
        plans = [plan]
        if world > 1:
            plans = [None] * world
            dist.all_gather_object(plans, plan)
        tmax = allreduce_max([float(rank + 1)], None, True)[0]
        if rank == 0:
            print(json.dumps({"n_gpus": world, "plans": plans, "max_over_ranks_check": tmax}))
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.sweep:
        run_sweep(args, rank, world, local_rank)
        return
    if args.fetch:
        if rank == 0:
            print(json.dumps(run_fetch(args, args.dev_idx)))
        return
    res = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick and not args.bf16:
        res["cpu_baseline"] = cpu_baseline(args, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

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
    ap.add_argument("--tp", type=int, default=2, help="--mode dptp: TP group size (world = DP x TP)")
    ap.add_argument("--fused-gather", action="store_true",
                    help="tp / dptp: all-gather fused into the combine epilogue (mla_combine_gather, symmetric memory)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--quick", action="store_true",
                    help="profiling runs: no clock-settle loop, no e2e leg, no cpu baseline")
    ap.add_argument("--mtp", type=int, default=1, help="query tokens per request per step (MTP, NEXT-1)")
    ap.add_argument("--fetch", action="store_true", help="time mla_kv_fetch_dequant over the workload cache")
    ap.add_argument("--bf16", action="store_true",
                    help="NEXT-2: the unquantized BF16 baseline (mla_decode_bf16, same skeleton) on the same workload")
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE.json configs[4]: DeepSeek-R1 shape over contexts 4K-128K x batch 1-512")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


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
    """dram bytes per decode launch from the committed ncu --set full summary, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(workload_key)
    return None if e is None else e.get("dram_bytes_per_launch")


# ------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2602_10718_b200 import dist as D
    from paper_2602_10718_b200 import ops, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = workload(args)
    B, H, L = w["batch"], w["heads"], w["context"]
    T = args.mtp
    # head partition: TP over the whole world, or over consecutive-rank TP groups (DP x TP)
    tp_world, t_idx, d_idx, tp_group = 1, 0, rank, None
    if args.mode == "tp":
        tp_world, t_idx, d_idx = world, rank, 0
    elif args.mode == "dptp":
        tp_world = args.tp
        d_idx, t_idx = D.dptp_coords(world, tp_world, rank)
        tp_group = D.dptp_groups(world, tp_world) if world > 1 else None
    n_dp = world // tp_world
    head0, head1 = D.tp_range(H, tp_world, t_idx)
    heads_local = head1 - head0
    scale = synth.DEFAULT_SOFTMAX_SCALE

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
        else:
            decode_fp8(qx, cache.kv_fp8, cache.kv_rope, cache.kv_scale, block_table, seq_lens, scale, ws)
    gathered, peer_ptrs = None, None
    if tp_world > 1 and args.fused_gather:
        if T > 1:
            raise SystemExit("--fused-gather supports mtp = 1")
        gathered, peer_ptrs = D.symmetric_gather_output((B, H, 512), tp_group or dist.group.WORLD, dev)
    elif tp_world > 1:
        gathered = torch.empty(tp_world, B, heads_local, 512, dtype=torch.bfloat16, device=dev)

    if peer_ptrs is not None:
        out = gathered[:, head0:head1]   # this rank's heads of the gathered result (e2e read-back)

    def combine_and_gather(out_t=None, lse_t=None):
        out_t = out if out_t is None else out_t
        lse_t = lse if lse_t is None else lse_t
        if peer_ptrs is not None:   # NEXT-4(c): peer stores from the combine epilogue + stream barrier
            ops.mla_combine_gather(ws, B, rows, peer_ptrs, t_idx, lse_t)
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

    def step(i=None):
        # a1: the T new tokens of every request land at positions L-T .. L-1 (same slots each step)
        for t in range(T):
            cache.append(new_cr[t][0], new_cr[t][1], block_table, seq_lens_t[t])
        if i is not None:
            ev_d0[i].record(stream)
        decode(q)
        if i is not None:
            ev_d1[i].record(stream)
        combine_and_gather()

    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    t_settle = time.time()
    while not args.quick and time.time() - t_settle < 1.0:        # keep the GPU loaded so clocks are sampled under load
        for _ in range(10):
            step()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(args.steps):
        step()          # no events between the kernels of the timed steps (an event record breaks the PDL overlap)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # per-launch decode time for the roofline: a second pass of the same steps with events
    # around each decode (plan + decode launches) on the launching stream
    for i in range(args.steps):
        step(i)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    dec_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev_d0, ev_d1)]))
    if world > 1:
        t = torch.tensor([ms, dec_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, dec_ms = float(t[0]), float(t[1])
    ms_step = ms / args.steps

    peak, peak_src = measured_peaks()
    bytes_per_token = 2 * (512 + 64) if args.bf16 else BYTES_PER_TOKEN
    kv_bytes = B * L * bytes_per_token
    dec_bytes = kv_bytes + B * rows * 576 * 2       # algorithmic bytes per decode launch
    achieved = dec_bytes / (dec_ms / 1e3) / 1e9
    tokens_per_step = B * T * n_dp
    if args.quick:
        return {"metric": METRIC, "value": round(tokens_per_step / (ms_step / 1e3), 1),
                "unit": "tokens/s", "ms_per_step": ms_step, "decode_ms": dec_ms, "quick": True,
                "batch": B, "heads": H, "context": L, "mtp": T,
                "roofline_frac": round(achieved / peak, 4), "achieved_gbs": round(achieved, 1), "clocks": clk}

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
    e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t[0])
    h2d = q_h.numel() * 2 + c_h.numel() * 2 + r_h.numel() * 2
    d2h = out_h.numel() * 2 + lse_h.numel() * 4

    # the same, pipelined the way a serving loop runs it: step i+1's inputs are copied in
    # (copy stream) and step i's result is read back (read-back stream) while step i
    # computes; double-buffered device inputs / outputs, every byte still crosses PCIe
    # inside the timed region
    cp_s, rb_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    din = [(torch.empty_like(q), torch.empty_like(new_c), torch.empty_like(new_r)) for _ in range(2)]
    dout = [(torch.empty_like(out) if peer_ptrs is None else out, torch.empty_like(lse)) for _ in range(2)]
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
        combine_and_gather(dout[k][0], dout[k][1])
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
    p_ms = p0.elapsed_time(p1)
    if world > 1:
        t = torch.tensor([p_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        p_ms = float(t[0])

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
        "scaling": "strong" if args.mode == "tp" else "weak",
        "vs_baseline": None,
        "dtype": "bf16 (NEXT-2 unquantized baseline; f32 accumulate)" if args.bf16 else "fp8e4m3 (f32 accumulate; bf16 RoPE)",
        "data": "synthetic (seeded MLA-like latent / RoPE distributions, random page permutation)",
        "config": {
            "workload": w["name"] + (" [BF16 baseline cache, NEXT-2]" if args.bf16 else ""), "batch_per_rank": B, "heads": H, "heads_per_rank": heads_local,
            "context": L, "page": 64, "kv_lora_rank": 512, "rope_dim": 64, "mtp": T,
            "parallelism": f"dp{n_dp}tp{tp_world}" + ("+fused-gather" if peer_ptrs is not None else ""),
            "l2": f"inputs larger than L2: KV {kv_bytes / 1e9:.2f} GB per rank vs 126 MB L2",
        },
        "roofline": {
            "bound": "hbm", "kernel": ("mla_decode_bf16" if args.bf16 else "mla_decode_fp8") + " (plan + decode launches)",
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": ncu_traffic(args.workload) if T == 1 and not args.bf16 else None, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": dec_bytes, "decode_ms": round(dec_ms, 4),
            "bytes_per_unit": f"{bytes_per_token} B per cached token + 1152 B per (request, query token, head) q row",
        },
        "e2e": {"value": round(tokens_per_step / (p_ms / args.steps / 1e3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "mode": "pipelined: H2D of step i+1 (pinned host -> device, copy stream) and D2H of step i "
                        "(read-back stream) overlap the compute of step i; double-buffered",
                "serial_value": round(tokens_per_step / (e_ms / args.steps / 1e3), 1)},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk,
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
    cores = len(os.sched_getaffinity(0))
    return {"value": round(n / t_tot, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} whole requests of the workload ({H} heads x {L} context): append of the new "
                      f"token + q-quant + O7 closed-form decode + combine, numpy fp64, {t_tot:.1f} s",
            "threads": cores}


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
    cores = len(os.sched_getaffinity(0))
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)",
        "data": "synthetic", "config": {"workload": w["name"], "batch_per_rank": w["batch"], "heads": H,
                                        "context": L, "page": 64, "parallelism": "cpu"},
        "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step = 1 whole request ({H} heads x {L} context) of the workload"},
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
            a.workload, a.batch, a.context, a.heads, a.quick = "dsr1", B, L, 128, True
            a.steps, a.warmup = max(5, min(args.steps, 20)), 3
            r = run_ours(a, rank, world, local_rank)
            pts.append({k: r[k] for k in ("batch", "context", "value", "ms_per_step", "decode_ms",
                                          "roofline_frac", "achieved_gbs")} | {"sm_mhz": r["clocks"]["sm_mhz"]})
            torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "sweep": "BASELINE.json configs[4] (DeepSeek-R1 shape, 128 heads)",
                          "unit": "tokens/s", "n_gpus": world, "points": pts}))


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)))
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.sweep:
        run_sweep(args, rank, world, local_rank)
        return
    if args.fetch:
        if rank == 0:
            print(json.dumps(run_fetch(args, local_rank)))
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

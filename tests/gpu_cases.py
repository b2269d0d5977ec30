"""Shared builders for the GPU parity tests: the same seeded synthetic inputs
go to the CUDA path (through the C ABI) and to the oracle; the two share no
arithmetic.  The KV cache is filled by the product append kernel on the GPU
and by oracle.snapmla.append_quant on the CPU, then compared byte-for-byte
(test_gpu_append) before any decode comparison uses it.
"""
import numpy as np
import torch

from oracle import snapmla as O
from paper_2602_10718_b200 import ops, synth

PAGE = 64


class Case:
    """B requests with lengths `lens`, H heads, random page permutation."""

    def __init__(self, lens, H, seed=0, dist="mla", extra_pages=3, softmax_scale=None, q_len=1):
        self.lens = np.asarray(lens, dtype=np.int64)
        self.B, self.H, self.q_len = len(lens), H, q_len
        self.scale = synth.DEFAULT_SOFTMAX_SCALE if softmax_scale is None else softmax_scale
        rng = np.random.default_rng(seed)
        self.bt, self.num_pages = synth.paged_layout(rng, self.lens, extra_pages=extra_pages)
        n_tok = int(self.lens.sum())
        c, r = synth.latent_tokens(rng, max(n_tok, 1), dist)
        self.c_kv, self.k_pe = c[:n_tok], r[:n_tok]              # bf16 CPU tensors
        if q_len == 1:
            self.q = synth.queries(rng, self.B * H, dist).reshape(self.B, H, 576)
        else:   # MTP: q [B, q_len, H, 576]
            self.q = synth.queries(rng, self.B * q_len * H, dist).reshape(self.B, q_len, H, 576)
        # flattened token -> (request, position) and its paged slot
        self.tok_req = np.repeat(np.arange(self.B), self.lens)
        self.tok_pos = np.concatenate([np.arange(L) for L in self.lens]) if n_tok else np.zeros(0, np.int64)
        self.tok_page = self.bt[self.tok_req, self.tok_pos // PAGE] if n_tok else np.zeros(0, np.int64)

    # ------------------------------------------------------------------ GPU
    def gpu_cache(self):
        dev = "cuda"
        cache = ops.PagedMLACache(self.num_pages, dev)
        n = len(self.tok_pos)
        if n:
            # one append launch: every token is a one-token "request" whose single
            # block-table entry is its page and whose post-append length puts it
            # at the right in-page row.
            bt_v = torch.from_numpy(self.tok_page.astype(np.int32)[:, None]).to(dev)
            sl_v = torch.from_numpy((self.tok_pos % PAGE + 1).astype(np.int32)).to(dev)
            cache.append(self.c_kv.to(dev), self.k_pe.to(dev), bt_v, sl_v)
        torch.cuda.synchronize()
        return cache

    def gpu_decode(self, cache, f32_out=False, workspace=None):
        dev = "cuda"
        bt = torch.from_numpy(self.bt).to(dev)
        sl = torch.from_numpy(self.lens.astype(np.int32)).to(dev)
        q = self.q.to(dev)
        out, lse = ops.decode_step(q, cache, bt, sl, self.scale, workspace=workspace, f32_out=f32_out)
        torch.cuda.synchronize()
        return out.float().cpu().numpy(), lse.cpu().numpy()

    # --------------------------------------------------------------- oracle
    def oracle_pools(self):
        pools = dict(kv_fp8=np.zeros((self.num_pages, 64, 512), np.uint8),
                     kv_rope=np.zeros((self.num_pages, 64, 64), np.uint16),
                     kv_scale=np.zeros((self.num_pages, 64), np.float32))
        n = len(self.tok_pos)
        if n:
            codes, sig, rope = O.append_quant(self.c_kv.float().numpy(), self.k_pe.float().numpy())
            slots = self.tok_page.astype(np.int64) * PAGE + self.tok_pos % PAGE
            pools["kv_fp8"].reshape(-1, 512)[slots] = codes
            pools["kv_rope"].reshape(-1, 64)[slots] = rope
            pools["kv_scale"].reshape(-1)[slots] = sig
        return pools

    def oracle_request_mtp(self, pools, b):
        """O7 per query token over its causally visible keys (reading R25)."""
        return O.decode_request_mtp(self.q[b].float().numpy(), pools, self.bt[b], int(self.lens[b]), self.scale)

    def oracle_request(self, pools, b, heads=None, which="o7", mx=False):
        L = int(self.lens[b])
        q = self.q[b].float().numpy()
        if heads is not None:
            q = q[heads]
        if which == "o8":
            sl = slice(int(self.lens[:b].sum()), int(self.lens[:b + 1].sum()))
            return O.attn_o8(q, self.c_kv[sl].float().numpy(), self.k_pe[sl].float().numpy(), self.scale)
        qc, sq, qr = O.q_quant(q)
        kc, sk, kr = O.gather_request(pools, self.bt[b], L)
        if which == "o6":
            return O.attn_o6(qc, sq, qr, kc, sk, kr, self.scale)
        if mx:   # NEXT-4(b) variant (test_gpu_mx.py)
            return O.decode_mx(qc, sq, qr, kc, sk, kr, self.scale)
        return O.decode_o7(qc, sq, qr, kc, sk, kr, self.scale)


def cache_to_numpy(cache):
    return dict(kv_fp8=cache.kv_fp8.cpu().numpy(),
                kv_rope=cache.kv_rope.view(torch.int16).cpu().numpy().view(np.uint16),
                kv_scale=cache.kv_scale.cpu().numpy())


def parity_stats(got, ref):
    d = np.abs(got.astype(np.float64) - ref)
    rms = float(np.sqrt(np.mean(ref ** 2)))
    return float(d.max() / rms), float(d.mean() / rms)

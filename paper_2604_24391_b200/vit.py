"""BASELINE config 4: the token cache in front of a ViT encoder (§8(f) #2).

The reference has no model; this module pins the semantics the
config describes and measures them.  The encoder is SigLIP-so400m shaped and
randomly initialised: patch 14 at 448 x 448 (1024 tokens), width 1152, MLP
4304 (GELU-tanh), 16 heads, 27 pre-LN blocks, bf16.  Its matmuls and
attention are library kernels (cuBLAS / SDPA); the FreqCache decision and the
hidden-state splice are this package's sm_100a kernels.

Two cached-step modes (``CachedEncoder.step``):

* ``"layer1"`` — the config's literal wording: the cache holds each token's
  patch-embedding state (layer 0) and first-block output (layer 1).  Only
  recomputed tokens go through the patch embedding and block 1 (queries =
  recomputed tokens; keys/values = all tokens, reused ones from the
  displacement-mapped layer-0 cache); the block-1 outputs are spliced with
  the cached ones and blocks 2..27 run on all tokens.  Savings are bounded by
  block 1's share of the encoder (~3.7 %).
* ``"subset"`` — the deployment-style reading: the cache holds final hidden
  states; recomputed tokens run the whole encoder attending among
  themselves, reused tokens take their (displacement-mapped) cached final
  state.  The recomputed tokens of all streams are packed without padding
  ([sum K_b, D] GEMMs, jagged-nested SDPA per stream), so the encoder work
  scales with the recompute ratio.

Both splice through ``fc_splice`` (bf16, bit copies) with the select's
``src_map``, and both report the cosine similarity of their output to a full
recompute of the same frame.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .engine import FreqCacheEngine, splice, splice_packed

try:  # variable-length attention for the packed subset mode (library kernel)
    from flash_attn import flash_attn_varlen_func as _flash_varlen
except Exception:  # noqa: BLE001 - optional dependency
    _flash_varlen = None


@dataclass(frozen=True)
class ViTConfig:
    image: int = 448
    patch: int = 14
    width: int = 1152
    mlp: int = 4304
    heads: int = 16
    layers: int = 27

    @property
    def tokens(self):
        return (self.image // self.patch) ** 2


class Block(torch.nn.Module):
    def __init__(self, c: ViTConfig):
        super().__init__()
        self.h = c.heads
        self.ln1 = torch.nn.LayerNorm(c.width)
        self.qkv = torch.nn.Linear(c.width, 3 * c.width)
        self.proj = torch.nn.Linear(c.width, c.width)
        self.ln2 = torch.nn.LayerNorm(c.width)
        self.fc1 = torch.nn.Linear(c.width, c.mlp)
        self.fc2 = torch.nn.Linear(c.mlp, c.width)

    def _heads(self, x):
        # works for dense [B, n, D] and jagged nested [B, j, D] tensors
        return x.unflatten(-1, (self.h, x.shape[-1] // self.h)).transpose(1, 2)

    def attn(self, xq, xkv, key_padding=None):
        """Attention with queries from xq and keys/values from xkv."""
        d = xq.shape[-1]
        wq, wk, wv = self.qkv.weight.split(d)
        bq, bk, bv = self.qkv.bias.split(d)
        q = self._heads(F.linear(xq, wq, bq))
        k = self._heads(F.linear(xkv, wk, bk))
        v = self._heads(F.linear(xkv, wv, bv))
        mask = None if key_padding is None else key_padding[:, None, None, :]
        o = F.scaled_dot_product_attention(q, k, v, attn_mask=mask)
        return self.proj(o.transpose(1, 2).flatten(-2))

    def forward(self, x, key_padding=None):
        y = self.ln1(x)
        x = x + self.attn(y, y, key_padding)
        return x + self.fc2(F.gelu(self.fc1(self.ln2(x)), approximate="tanh"))

    def forward_packed(self, x, offsets, max_len):
        """Block over variable-length token sets packed as [T, D] (stream b's
        tokens at rows offsets[b] .. offsets[b+1]); attention stays within a
        stream: flash-attention varlen (library kernel) on [T, heads, hd],
        or jagged nested tensors through SDPA where flash_attn is absent."""
        y = self.ln1(x)
        d = x.shape[-1]
        hd = d // self.h
        q, k, v = (t.unflatten(-1, (self.h, hd)) for t in
                   F.linear(y, self.qkv.weight, self.qkv.bias).split(d, dim=-1))
        if _flash_varlen is not None and x.dtype in (torch.float16, torch.bfloat16):
            cu = offsets.to(torch.int32)
            o = _flash_varlen(q.contiguous(), k.contiguous(), v.contiguous(), cu, cu, max_len, max_len)
        else:
            def nj(t):
                return torch.nested.nested_tensor_from_jagged(t, offsets).transpose(1, 2)

            o = F.scaled_dot_product_attention(nj(q), nj(k), nj(v)).transpose(1, 2).values()
        x = x + self.proj(o.flatten(-2))
        return x + self.fc2(F.gelu(self.fc1(self.ln2(x)), approximate="tanh"))

    def forward_subset(self, xq, xkv):
        """Block output for query tokens xq given all tokens' inputs xkv."""
        x = xq + self.attn(self.ln1(xq), self.ln1(xkv))
        return x + self.fc2(F.gelu(self.fc1(self.ln2(x)), approximate="tanh"))


class ViT(torch.nn.Module):
    def __init__(self, c: ViTConfig = ViTConfig(), seed=0):
        super().__init__()
        self.c = c
        g = torch.Generator().manual_seed(seed)
        self.embed = torch.nn.Linear(3 * c.patch * c.patch, c.width)
        self.pos = torch.nn.Parameter(torch.zeros(c.tokens, c.width))
        self.blocks = torch.nn.ModuleList(Block(c) for _ in range(c.layers))
        self.ln = torch.nn.LayerNorm(c.width)
        with torch.no_grad():
            for p in self.parameters():
                if p.dim() >= 2:
                    p.copy_(torch.randn(p.shape, generator=g) * 0.02)

    def patches(self, frames):
        """[B, H, W, 3] -> [B, N, 3*P*P] row-major patches."""
        b, h, w, _ = frames.shape
        p = self.c.patch
        x = frames.view(b, h // p, p, w // p, p, 3).permute(0, 1, 3, 2, 4, 5)
        return x.reshape(b, (h // p) * (w // p), p * p * 3)

    def embed_tokens(self, patches, idx=None):
        pos = self.pos if idx is None else self.pos[idx]
        return self.embed(patches) + pos

    def forward(self, frames):
        x = self.embed_tokens(self.patches(frames).to(self.embed.weight.dtype))
        for blk in self.blocks:
            x = blk(x)
        return self.ln(x)


def _gather_rows(x, idx):
    """x [B, N, D], idx [B, K] (-1 padded) -> [B, K, D] (padding rows = 0)."""
    safe = idx.clamp_min(0).long()
    out = torch.gather(x, 1, safe[..., None].expand(-1, -1, x.shape[-1]))
    return out * (idx >= 0)[..., None].to(out.dtype)


class CachedEncoder:
    """Batched token-cache encoder over B streams (select + partial ViT + splice)."""

    def __init__(self, model: ViT, batch: int, mode: str = "layer1", device="cuda", group: int = 0):
        if mode not in ("layer1", "subset"):
            raise ValueError(mode)
        c = model.c
        self.m, self.mode, self.B, self.group = model, mode, batch, (group or batch)
        self.engine = FreqCacheEngine(batch, c.image, c.image, c.patch, fmt="rgb", device=device)
        n, d = c.tokens, c.width
        dt = next(model.parameters()).dtype
        self.h1 = torch.zeros((2, batch, n, d), dtype=dt, device=device)   # cached layer-1 / final
        self.h0 = torch.zeros((2, batch, n, d), dtype=dt, device=device)   # cached layer-0 (layer1 mode)
        self.ages = torch.zeros((2, batch, n), dtype=torch.int64, device=device)
        self.cur = 0

    @torch.no_grad()
    def step(self, frames, cfg, refresh_shift=None):
        """One decision + cached encoder step; returns final hidden states."""
        m, B = self.m, self.B
        out = self.engine.select(frames, cfg, refresh_shift=refresh_shift)
        rec = out.recompute_idx                       # [B, N] row-major, -1 padded
        kmax = int((rec >= 0).sum(dim=1).max().item())
        # pad the recompute batch to a bucket of 128 so GEMM / attention plans
        # are reused across steps (the -1 rows are masked out)
        kpad = min(rec.shape[1], max(128, -(-kmax // 128) * 128))
        rec = rec[:, :kpad]
        valid = rec >= 0
        patches = m.patches(frames.to(next(m.parameters()).dtype))
        p_rec = _gather_rows(patches, rec)
        x0 = m.embed_tokens(p_rec, rec.clamp_min(0).long())      # [B, K, D]
        i, o = self.cur, 1 - self.cur
        if self.mode == "layer1":
            # layer-0 states of all tokens: reused from the shifted cache, fresh for recomputed
            splice(out.src_map, self.h0[i], self.ages[i], x0.contiguous(), self.h0[o], self.ages[o],
                   compact=True)
            x1 = m.blocks[0].forward_subset(x0, self.h0[o])
            splice(out.src_map, self.h1[i], self.ages[i], x1.contiguous(), self.h1[o], self.ages[o],
                   compact=True)
            x = self.h1[o]
            for blk in m.blocks[1:]:
                x = blk(x)
            y = m.ln(x)
        else:
            # recomputed tokens of all streams packed stream-major (rec is
            # front-packed per stream), no padding
            counts = valid.sum(dim=1)
            offsets = torch.zeros(B + 1, dtype=torch.int64, device=rec.device)
            offsets[1:] = torch.cumsum(counts, 0)
            x = x0[valid]                                   # [sum K_b, D]
            if x.shape[0] == 0:
                packed = x0.new_zeros((1, x0.shape[-1]))
            else:
                seg = torch.unique_consecutive(offsets)     # streams with no recomputed token drop out
                max_len = int(counts.max().item())
                for blk in m.blocks:
                    x = blk.forward_packed(x, seg, max_len)
                packed = m.ln(x)
            splice_packed(out.src_map, self.h1[i], self.ages[i], packed, offsets[:B].contiguous(),
                          self.h1[o], self.ages[o])
            y = self.h1[o]
        self.cur = o
        return y, out

    def flops_per_frame(self, n_tokens):
        """Approximate encoder FLOPs for n tokens (matmuls + attention)."""
        c = self.m.c
        d, f = c.width, c.mlp
        per_layer = 2 * n * (3 * d * d + d * d + 2 * d * f) + 4 * n * n * d
        return c.layers * per_layer + 2 * n * 3 * c.patch * c.patch * d


def cosine(a, b):
    a = a.float().flatten(1)
    b = b.float().flatten(1)
    return (a * b).sum(1) / (a.norm(dim=1) * b.norm(dim=1)).clamp_min(1e-30)

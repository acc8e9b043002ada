"""BASELINE config 4: the token cache in front of a ViT encoder (§8(f) #2).

The reference has no model; this module pins the semantics the
config describes and measures them.  The encoder is SigLIP-so400m shaped and
randomly initialised: patch 14 at 448 x 448 (1024 tokens), width 1152, MLP
4304 (GELU-tanh), 16 heads, 27 pre-LN blocks, bf16.  Its matmuls and
attention are library kernels (cuBLAS / SDPA); the FreqCache decision and the
hidden-state splice are this package's sm_100a kernels.

Two cached-step modes (``CachedEncoder.step``):

* ``"layer1"`` — the config's literal wording: only recomputed tokens go
  through the patch embedding and the first block; the cache holds each
  token's first-block keys / values and output.  Queries = recomputed
  tokens; keys/values = all tokens (reused ones from the displacement-mapped
  K/V cache); the first-block outputs are spliced with the cached ones and
  blocks 2..27 run on all tokens.  Savings are bounded by the first block's
  share of the encoder (~3.7 %).
* ``"subset"`` — the deployment-style reading: the cache holds final hidden
  states; recomputed tokens run the whole encoder attending among
  themselves, reused tokens take their (displacement-mapped) cached final
  state.  The recomputed tokens of all streams are packed without padding
  ([sum K_b, D] GEMMs; attention within each stream by cuDNN's ragged
  kernel, else flash-attention varlen, else jagged-nested SDPA), so the
  encoder work scales with the recompute ratio; the bf16 step replays from a
  CUDA graph per packed-row bucket.

Both splice through ``fc_splice`` (bf16, bit copies, device-side bounds
check) with the select's ``src_map``, and both report the cosine similarity
of their output to a full recompute of the same frame.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .engine import FreqCacheEngine, gather_patches, splice, splice_packed

try:  # variable-length attention for the packed subset mode (library kernel)
    from flash_attn import flash_attn_varlen_func as _flash_varlen
except Exception:  # noqa: BLE001 - optional dependency
    _flash_varlen = None
try:  # cuDNN ragged attention through flashinfer's wrapper (library kernel)
    from flashinfer.prefill import cudnn_batch_prefill_with_kv_cache as _cudnn_ragged
except Exception:  # noqa: BLE001 - optional dependency
    _cudnn_ragged = None


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

    def forward_packed(self, x, offsets, max_len, ragged=None):
        """Block over variable-length token sets packed as [T, D] (stream b's
        tokens at rows offsets[b] .. offsets[b+1]); attention stays within a
        stream: ``ragged(q, k, v)`` (cuDNN ragged attention on contiguous
        [T, heads, hd] q / k / v) when given, else flash-attention varlen
        (library kernel) on strided views, else jagged nested tensors through
        SDPA where flash_attn is absent."""
        y = self.ln1(x)
        d = x.shape[-1]
        hd = d // self.h
        if ragged is not None:
            # three projections, so q, k and v are each contiguous (the
            # ragged kernel takes token-contiguous rows)
            w, bias = self.qkv.weight.split(d), self.qkv.bias.split(d)
            q, k, v = (F.linear(y, w[j], bias[j]).view(-1, self.h, hd) for j in range(3))
            o = ragged(q, k, v)
            x = x + self.proj(o.reshape(-1, d))
            return x + self.fc2(F.gelu(self.fc1(self.ln2(x)), approximate="tanh"))
        q, k, v = (t.unflatten(-1, (self.h, hd)) for t in
                   F.linear(y, self.qkv.weight, self.qkv.bias).split(d, dim=-1))
        if _flash_varlen is not None and x.dtype in (torch.float16, torch.bfloat16):
            cu = offsets.to(torch.int32)
            # q / k / v stay strided views of the QKV output (unit stride in
            # the head dimension is all the kernel needs): no copies
            o = _flash_varlen(q, k, v, cu, cu, max_len, max_len)
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


class CachedEncoder:
    """Batched token-cache encoder over B streams (select + partial ViT + splice).

    Host synchronisation: the only values the host needs (the recompute
    count of every stream, which sizes the recompute bucket and the packed
    batch) come from the select's results record.  The select of the next
    step can be issued ahead (``step(..., next_frames=...)``) on a side
    stream, so by the time the host reads those counts the select has long
    finished and the device queue still holds the previous step's encoder
    blocks — the host waits on the select's event, never on the encoder.

    Recomputed tokens of all streams are packed without padding ([sum K_b, D]
    rows), so the partial work scales with the recompute ratio of each
    stream rather than the worst stream's.

    ``layer1`` caches every token's block-0 q | k | v row and block-0 output
    (displacement-mapped like the tokens): recomputed tokens run the patch
    embedding, LN and the QKV projection, their fresh q | k | v rows are
    spliced into the cache (``fc_splice_packed``, one 3D-wide row per token),
    one dense attention runs over all tokens of each stream (library SDPA:
    cheaper on B200 than a variable-length kernel for the recomputed queries
    only) and only the recomputed rows go on through the projection and the
    MLP; the block-0 outputs are spliced with the cached ones and blocks
    1..26 run on every token, replayed from a CUDA graph (static shapes).
    Reused tokens skip the embedding, block-0 QKV, projection and MLP.
    """

    def __init__(self, model: ViT, batch: int, mode: str = "layer1", device="cuda", group: int = 0,
                 graphs: bool = True):
        if mode not in ("layer1", "subset"):
            raise ValueError(mode)
        c = model.c
        self.m, self.mode, self.B, self.group = model, mode, batch, (group or batch)
        self.device = torch.device(device)
        self.engine = FreqCacheEngine(batch, c.image, c.image, c.patch, fmt="rgb", device=device)
        n, d = c.tokens, c.width
        dt = next(model.parameters()).dtype
        self.h1 = torch.zeros((2, batch, n, d), dtype=dt, device=device)   # cached block-0 output / final
        if mode == "layer1":
            # cached block-0 q | k | v rows of every token (one 3D-wide row per token)
            self.qkv0 = torch.zeros((2, batch, n, 3 * d), dtype=dt, device=device)
        self.tail_graphs = {} if (graphs and mode == "layer1") else None
        self._tail_out = {}
        # layer1 with graphs: the packed block-0 work of a step is replayed
        # from a CUDA graph per (row bucket, cache buffer); its per-step inputs
        # are copied into static buffers first
        self.b0_graphs = {} if self.tail_graphs is not None else None
        # subset with graphs: the whole packed encoder of a step is replayed
        # from a CUDA graph per (row bucket, cache buffer) — 27 blocks of
        # eager launches would leave the GPU waiting on the host
        # (flash-attention varlen, bf16 / fp16, takes the zero-length and
        # padding segments inside a graph; other dtypes run eagerly)
        self.sub_graphs = ({} if (graphs and mode == "subset" and _flash_varlen is not None
                                  and dt in (torch.float16, torch.bfloat16)) else None)
        # graphed subset attention: cuDNN ragged attention (flashinfer's
        # wrapper) where available, 2.2x faster than flash-attention varlen on
        # B200 at head dim 72 (scripts/attn_probe2.py); FC_VIT_ATTN=fa2 keeps
        # flash-attention
        self.cudnn_attn = (self.sub_graphs is not None and _cudnn_ragged is not None
                           and os.environ.get("FC_VIT_ATTN", "cudnn") == "cudnn")
        if self.cudnn_attn:
            self.attn_ws = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        nb = batch * n
        self.bucket = max(64, min(1024, -(-nb // 16 // 64) * 64))   # ~16 row buckets
        if self.b0_graphs is not None or self.sub_graphs is not None:
            self.st_frames = torch.zeros((batch, c.image, c.image, 3), dtype=torch.float32, device=device)
            self.st_src = torch.zeros((batch, n), dtype=torch.int32, device=device)
            self.st_rec = torch.zeros((batch, n), dtype=torch.int32, device=device)
            self.st_offsets = torch.zeros(batch + 1, dtype=torch.int64, device=device)
            self._pool = torch.cuda.graph_pool_handle()
        self.ages = torch.zeros((2, batch, n), dtype=torch.int64, device=device)
        self.scratch_ages = torch.zeros((batch, n), dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)      # splice bounds flag
        self.cur = 0
        # select results double-buffered; counts to the host through pinned memory
        self.outs = [self.engine.new_output(), self.engine.new_output()]
        self.sel_stream = torch.cuda.Stream(self.device)
        self.select_on_main = os.environ.get("FC_VIT_SELECT_MAIN") == "1"   # diagnostics knob
        self.debug_marks = None   # diagnostics: a list receives per-step (start, block 0 done, tail done) events
        self.host_counts = [torch.zeros(batch, dtype=torch.int32).pin_memory() for _ in range(2)]
        # packed-row offsets per select slot, built on the device (no
        # per-step pinned allocations: those can synchronise the device)
        self.offsets = [torch.zeros(batch + 1, dtype=torch.int64, device=device) for _ in range(2)]
        self.sel_done = [torch.cuda.Event(), torch.cuda.Event()]
        self.pending = None   # (frames tensor, slot) of a select issued ahead
        self.k = 0
        if self.tail_graphs is not None:   # capture every graph up front (fresh, all-zero caches)
            with torch.no_grad():
                for o in (0, 1):
                    self._tail(o)
        self.prepare_graphs()

    def _issue_select(self, frames, cfg, refresh_shift):
        """Select on the side stream (in stream order with every earlier
        select: the spectrum state); recompute counts -> pinned host."""
        slot = self.k
        self.k ^= 1
        main = torch.cuda.current_stream(self.device)
        st = main if self.select_on_main else self.sel_stream
        if st is not main:
            st.wait_stream(main)                 # frames / earlier consumers of this slot
        with torch.cuda.stream(st):
            out = self.engine.select(frames, cfg, out=self.outs[slot], refresh_shift=refresh_shift)
            kf = out.results.view(torch.int32)[:, 6]           # fc_stream_result.k_final
            rec = self.m.c.tokens - kf                          # recomputed tokens per stream
            torch.cumsum(rec, 0, out=self.offsets[slot][1:])
            self.host_counts[slot].copy_(rec, non_blocking=True)
            self.sel_done[slot].record(st)
        return slot

    @torch.no_grad()
    def step(self, frames, cfg, refresh_shift=None, next_frames=None):
        """One decision + cached encoder step; returns final hidden states.
        ``next_frames``: the next step's frames, whose select is then issued
        ahead on the side stream (it needs only the frames and this step's
        spectrum state)."""
        m, B = self.m, self.B
        if self.pending is not None and self.pending[0] is frames:
            slot = self.pending[1]
        else:
            slot = self._issue_select(frames, cfg, refresh_shift)
        self.pending = None
        main = torch.cuda.current_stream(self.device)
        main.wait_event(self.sel_done[slot])
        marks = self.debug_marks
        if marks is not None:
            marks.append([torch.cuda.Event(enable_timing=True) for _ in range(3)])
            marks[-1][0].record(main)
        out = self.outs[slot]
        self.sel_done[slot].synchronize()        # the select only, not the encoder queue
        counts = self.host_counts[slot].tolist()
        kmax = max(counts)
        n = m.c.tokens
        dt = next(m.parameters()).dtype
        i, o = self.cur, 1 - self.cur
        # recomputed tokens of all streams packed stream-major without
        # padding (stream b's k-th recomputed token, row-major, at row
        # offsets[b] + k — the fc_splice_packed layout); shapes from the host
        # counts, so nothing here waits on the device
        total = sum(counts)
        offsets = self.offsets[slot]
        if self.mode == "layer1" and self.b0_graphs is not None and total:
            self.st_frames.copy_(frames)
            self.st_src.copy_(out.src_map)
            self.st_rec.copy_(out.recompute_idx)
            self.st_offsets.copy_(offsets)
            tp = -(-total // self.bucket) * self.bucket
            self._block0_graph(tp, o).replay()
            self._prefetch(next_frames, cfg, refresh_shift)
            if marks is not None:
                marks[-1][1].record(main)
            y = self._tail(o)
            if marks is not None:
                marks[-1][2].record(main)
            self.cur = o
            return y, out
        if total:
            sid = torch.repeat_interleave(torch.arange(B, device=self.device), offsets[1:] - offsets[:-1],
                                          output_size=total)
            pos = torch.arange(total, device=self.device) - offsets[sid]
            tok = out.recompute_idx.view(-1).index_select(0, sid * n + pos).long()
            flat = sid * n + tok
            x = m.embed(self._embed_input(frames, flat, dt)) + m.pos.index_select(0, tok)   # [T, D] layer 0
        if self.mode == "layer1":
            blk = m.blocks[0]
            d = m.c.width
            # fresh block-0 q | k | v rows of the recomputed tokens, spliced
            # into the cache of all tokens (reused rows displacement-mapped)
            qkv = (F.linear(blk.ln1(x), blk.qkv.weight, blk.qkv.bias) if total
                   else torch.zeros((1, 3 * d), dtype=dt, device=self.device))
            splice_packed(out.src_map, self.qkv0[i], self.ages[i], qkv, offsets[:B].contiguous(), self.qkv0[o],
                          self.scratch_ages, status=self.status)
            if total:
                # attention over every token of the stream (one dense SDPA);
                # only the recomputed tokens' rows are kept
                q, k, v = (blk._heads(t) for t in self.qkv0[o].split(d, dim=-1))
                att = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B * n, d)
                x = x + blk.proj(att.index_select(0, flat))
                x1 = x + blk.fc2(F.gelu(blk.fc1(blk.ln2(x)), approximate="tanh"))
            else:
                x1 = torch.zeros((1, d), dtype=dt, device=self.device)
            splice_packed(out.src_map, self.h1[i], self.ages[i], x1, offsets[:B].contiguous(), self.h1[o],
                          self.ages[o], status=self.status)
            self._prefetch(next_frames, cfg, refresh_shift)
            if marks is not None:
                marks[-1][1].record(main)
            y = self._tail(o)
            if marks is not None:
                marks[-1][2].record(main)
        elif self.sub_graphs is not None and total:
            self.st_frames.copy_(frames)
            self.st_src.copy_(out.src_map)
            self.st_rec.copy_(out.recompute_idx)
            self.st_offsets.copy_(offsets)
            tp = -(-total // self.bucket) * self.bucket
            self._subset_graph(tp, o).replay()
            self._prefetch(next_frames, cfg, refresh_shift)
            y = self.h1[o]
        else:
            # the whole packed encoder follows: the next select goes beside it
            self._prefetch(next_frames, cfg, refresh_shift)
            if total == 0:
                packed = torch.zeros((1, m.c.width), dtype=dt, device=self.device)
            else:
                # segment bounds of the streams that recompute anything (sizes
                # known on the host, so no device sync)
                nz = sum(1 for cnt in counts if cnt > 0)
                keep = torch.nonzero_static(offsets[1:] > offsets[:-1], size=nz).flatten()
                seg = torch.cat([offsets[:1], offsets[1:][keep]])
                for blk in m.blocks:
                    x = blk.forward_packed(x, seg, kmax)
                packed = m.ln(x)
            splice_packed(out.src_map, self.h1[i], self.ages[i], packed, offsets[:B].contiguous(),
                          self.h1[o], self.ages[o], status=self.status)
            y = self.h1[o]
        self.cur = o
        return y, out

    def _prefetch(self, next_frames, cfg, refresh_shift):
        """Issue the next step's select once this step's partial (block-0 /
        packed) work is enqueued: it then runs beside the long static tail
        instead of competing with the next step's block-0 work."""
        if next_frames is not None:
            self.pending = (next_frames, self._issue_select(next_frames, cfg, refresh_shift))

    def _block0_static(self, tp, o):
        """Packed block-0 work of one step on the static buffers, for tp
        (>= the step's recomputed rows) packed rows: gathers, embedding, LN,
        QKV, the q|k|v splice, dense attention, projection + MLP for the
        recomputed rows, the block-0 output splice.  Rows past the step's
        count compute throw-away values that no splice reads."""
        m, B = self.m, self.B
        n, d = m.c.tokens, m.c.width
        dt = next(m.parameters()).dtype
        i = 1 - o
        blk = m.blocks[0]
        offsets = self.st_offsets
        ar = torch.arange(tp, device=self.device)
        sid = torch.searchsorted(offsets[1:], ar, right=True).clamp_(max=B - 1)
        pos = (ar - offsets[sid]).clamp_(0, n - 1)
        tok = self.st_rec.view(-1).index_select(0, sid * n + pos).long().clamp_(min=0)
        flat = sid * n + tok                                     # token b * N + p of each packed row
        x = m.embed(self._embed_input(self.st_frames, flat, dt)) + m.pos.index_select(0, tok)
        qkv = F.linear(blk.ln1(x), blk.qkv.weight, blk.qkv.bias)
        splice_packed(self.st_src, self.qkv0[i], self.ages[i], qkv, offsets[:B], self.qkv0[o], self.scratch_ages,
                      status=self.status)
        q, k, v = (blk._heads(t) for t in self.qkv0[o].split(d, dim=-1))   # reused rows' q: never read back
        att = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B * n, d)
        x = x + blk.proj(att.index_select(0, flat))
        x1 = x + blk.fc2(F.gelu(blk.fc1(blk.ln2(x)), approximate="tanh"))
        splice_packed(self.st_src, self.h1[i], self.ages[i], x1, offsets[:B], self.h1[o], self.ages[o],
                      status=self.status)

    def _subset_static(self, tp, o):
        """The subset step on the static buffers for tp (>= the step's
        recomputed rows) packed rows: gathers, embedding, every block over
        the packed rows (attention within each stream's segment; the rows
        past the step's count form one extra segment of their own), final
        LN, the splice into cache buffer o.  Padding rows compute throw-away
        values that no splice reads."""
        m, B = self.m, self.B
        n = m.c.tokens
        dt = next(m.parameters()).dtype
        i = 1 - o
        offsets = self.st_offsets
        ar = torch.arange(tp, device=self.device)
        sid = torch.searchsorted(offsets[1:], ar, right=True).clamp_(max=B - 1)
        pos = (ar - offsets[sid]).clamp_(0, n - 1)
        tok = self.st_rec.view(-1).index_select(0, sid * n + pos).long().clamp_(min=0)
        flat = sid * n + tok
        x = m.embed(self._embed_input(self.st_frames, flat, dt)) + m.pos.index_select(0, tok)
        # segments: the B streams (empty ones have zero length), then padding
        seg = torch.cat([offsets, torch.full((1,), tp, dtype=offsets.dtype, device=self.device)])
        ragged = None
        if self.cudnn_attn:
            h = m.c.heads
            hd = m.c.width // h
            lens = (seg[1:] - seg[:-1]).to(torch.int32).view(-1, 1, 1, 1)
            rows = (seg * (h * hd)).to(torch.int32).view(-1, 1, 1, 1)     # element offsets of each segment
            ws, mx = self.attn_ws, max(n, self.bucket)

            def ragged(q, k, v):
                return _cudnn_ragged(q, k, v, hd ** -0.5, ws, max_token_per_sequence=mx, max_sequence_kv=mx,
                                     actual_seq_lens_q=lens, actual_seq_lens_kv=lens, causal=False,
                                     return_lse=False, batch_offsets_q=rows, batch_offsets_o=rows,
                                     batch_offsets_k=rows, batch_offsets_v=rows, is_cuda_graph_compatible=True)[0]
        for blk in m.blocks:
            x = blk.forward_packed(x, seg, max(n, self.bucket), ragged)
        packed = m.ln(x)
        splice_packed(self.st_src, self.h1[i], self.ages[i], packed, offsets[:B], self.h1[o], self.ages[o],
                      status=self.status)

    def _subset_graph(self, tp, o):
        key = (tp, o)
        g = self.sub_graphs.get(key)
        if g is None:
            st = torch.cuda.Stream(self.device)
            st.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(st):          # warm-up outside capture (library plans)
                self._subset_static(tp, o)
            torch.cuda.current_stream(self.device).wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self._pool):
                self._subset_static(tp, o)
            self.sub_graphs[key] = g
        return g

    def _embed_input(self, frames, flat, dt):
        """Patch pixels of the packed tokens: gathered straight from fp32 RGB
        frames in bf16 (``fc_gather_patches``), else through torch."""
        c = self.m.c
        if dt == torch.bfloat16 and frames.dtype == torch.float32 and frames.is_contiguous():
            return gather_patches(frames, c.patch, flat)
        return self.m.patches(frames.to(dt)).reshape(-1, 3 * c.patch * c.patch).index_select(0, flat)

    def _block0_graph(self, tp, o):
        key = (tp, o)
        g = self.b0_graphs.get(key)
        if g is None:
            # warm-up (library plans) outside capture; harmless before the
            # first step (prepare_graphs), when the caches hold no state yet
            st = torch.cuda.Stream(self.device)
            st.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(st):
                self._block0_static(tp, o)
            torch.cuda.current_stream(self.device).wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self._pool):
                self._block0_static(tp, o)
            self.b0_graphs[key] = g
        return g

    def prepare_graphs(self):
        """Capture every bucket graph up front (no capture inside a timed
        loop); the caches hold no state yet, so the warm-up runs are
        harmless."""
        make = self._block0_graph if self.b0_graphs is not None else (
            self._subset_graph if self.sub_graphs is not None else None)
        if make is None:
            return
        with torch.no_grad():
            nb = self.B * self.m.c.tokens
            for tp in range(self.bucket, -(-nb // self.bucket) * self.bucket + 1, self.bucket):
                for o in (0, 1):
                    make(tp, o)
            self.h1.zero_()
            self.ages.zero_()
            self.status.zero_()

    def _tail(self, o):
        """Blocks 1.. and the final LN on every token of cache buffer o —
        static shapes, so captured once per buffer in a CUDA graph and
        replayed (no per-kernel host launches)."""
        m = self.m
        if self.tail_graphs is None:
            x = self.h1[o]
            for blk in m.blocks[1:]:
                x = blk(x)
            return m.ln(x)
        g = self.tail_graphs.get(o)
        if g is None:
            st = torch.cuda.Stream(self.device)
            st.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(st):          # warm-up outside capture (library plans)
                x = self.h1[o]
                for blk in m.blocks[1:]:
                    x = blk(x)
                m.ln(x)
            torch.cuda.current_stream(self.device).wait_stream(st)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                x = self.h1[o]
                for blk in m.blocks[1:]:
                    x = blk(x)
                self._tail_out[o] = m.ln(x)
            self.tail_graphs[o] = g
        g.replay()
        return self._tail_out[o]

    def check(self):
        """Raise AssertionError if a splice met an out-of-bounds source."""
        from .engine import check_status
        try:
            check_status(self.status, "CachedEncoder splice")
        finally:
            self.status.zero_()

    def flops_per_frame(self, n_tokens):
        """Approximate encoder FLOPs for n tokens (matmuls + attention)."""
        c = self.m.c
        d, f = c.width, c.mlp
        per_layer = 2 * n_tokens * (3 * d * d + d * d + 2 * d * f) + 4 * n_tokens * n_tokens * d
        return c.layers * per_layer + 2 * n_tokens * 3 * c.patch * c.patch * d


class GraphedViT:
    """Full recompute through one CUDA graph (static [B, H, W, 3] input
    buffer): the baseline the cached step is compared with, launched the same
    way as the cached step's static tail."""

    def __init__(self, model: ViT, batch: int, device="cuda"):
        c = model.c
        self.m = model
        self.x = torch.zeros((batch, c.image, c.image, 3), dtype=torch.float32, device=device)
        st = torch.cuda.Stream(device)
        st.wait_stream(torch.cuda.current_stream(device))
        with torch.no_grad(), torch.cuda.stream(st):
            model(self.x)
        torch.cuda.current_stream(device).wait_stream(st)
        self.g = torch.cuda.CUDAGraph()
        with torch.no_grad(), torch.cuda.graph(self.g):
            self.y = model(self.x)

    def __call__(self, frames):
        self.x.copy_(frames)
        self.g.replay()
        return self.y


def cosine(a, b):
    a = a.float().flatten(1)
    b = b.float().flatten(1)
    return (a * b).sum(1) / (a.norm(dim=1) * b.norm(dim=1)).clamp_min(1e-30)

"""Decision serialization from device outputs.

Same on-disk formats as the reference (records.py:12-77, frameio.py:91-105,
188-219): JSON Lines decisions, a fixed-header metrics CSV and one
patch-resolution PGM mask per step.  Mask images are rendered on the GPU
from the select outputs (``render_masks``: reused 255, edge-forced
recompute 128, other 0, flushed steps all 0) and only the finished bytes
are copied to the host.  Outputs are deterministic, so reruns are
byte-identical (the reference's acceptance criterion 7).
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np
import torch

METRICS_HEADER = ["step", "reuse_ratio", "sim_freq", "entropy", "alpha", "latency_model_ms"]
MASK_REUSED, MASK_EDGE_RECOMPUTE, MASK_RECOMPUTE = 255, 128, 0


def decision_record(d, include_timings=False):
    """CacheDecision -> the reference's JSONL dict (records.py:16-43)."""
    rec = {
        "step": d.step,
        "flushed": d.flushed,
        "sim_freq": d.sim_freq,
        "displacement": {"di": d.displacement.di, "dj": d.displacement.dj,
                         "di_p": d.displacement.di_patches, "dj_p": d.displacement.dj_patches},
        "entropy": {"raw": d.entropy.raw, "normalized": d.entropy.normalized},
        "alpha": d.alpha_t,
        "k_reuse": d.k_reuse,
        "k_candidate": d.k_candidate,
        "k_final": d.k_final,
        "reuse_set": list(d.reuse_set),
        "grid": {"rows": d.rows, "cols": d.cols},
        "refresh_set": list(d.refresh_set),
        "diagnostic": d.diagnostic,
    }
    if include_timings:
        rec["timings_us"] = {k: int(v) for k, v in d.timings_us.items()}
    return rec


def write_decisions_jsonl(path, decisions, include_timings=False):
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for d in decisions:
            fh.write(json.dumps(decision_record(d, include_timings)))
            fh.write("\n")


def read_decisions_jsonl(path):
    with open(path, "r", encoding="utf-8") as fh:
        return [json.loads(line) for line in fh if line.strip()]


def metrics_rows(report):
    return [[d.step, d.k_final / report.n_tokens, d.sim_freq, d.entropy.normalized, d.alpha_t,
             r.latency_model_ms] for d, r in zip(report.decisions, report.step_reports)]


def write_metrics_csv(path, report):
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(METRICS_HEADER)
        w.writerows(metrics_rows(report))


def write_pgm(path, img_u8):
    a = np.ascontiguousarray(img_u8, dtype=np.uint8)
    if a.ndim != 2:
        raise ValueError(f"image must be 2D, got shape {a.shape}")
    h, w = a.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{w} {h}\n255\n".encode("ascii"))
        fh.write(a.tobytes())


def render_masks(out, engine=None):
    """Device mask images [B, rows, cols] uint8 from a SelectResult."""
    from . import _native as nat
    from .engine import _ptr, _stream
    B, N = out.reuse_mask.shape
    img = torch.empty((B, N), dtype=torch.uint8, device=out.reuse_mask.device)
    nat.check(nat.lib().fc_render_masks(int(B), int(N), _ptr(out.results), _ptr(out.reuse_mask),
                                        _ptr(out.refresh_mask), _ptr(img), _stream(img.device)),
              "fc_render_masks")
    if engine is not None:
        return img.view(B, engine.rows, engine.cols)
    return img


def export_masks(decisions_or_images, out_dir, steps=None):
    """One PGM per step (frameio.py:197-219).  Accepts CacheDecisions / JSONL
    dicts (rendered on the host from their index sets, for files written by
    earlier runs) or a device/host image batch from ``render_masks`` plus the
    step numbers."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    paths = []
    if isinstance(decisions_or_images, torch.Tensor):
        imgs = decisions_or_images.cpu().numpy()
        steps = list(range(len(imgs))) if steps is None else list(steps)
        for img, st in zip(imgs, steps):
            p = out_dir / f"step_{int(st):05d}.pgm"
            write_pgm(p, img)
            paths.append(p)
        return paths
    for d in decisions_or_images:
        rec = d if isinstance(d, dict) else decision_record(d)
        rows, cols = rec["grid"]["rows"], rec["grid"]["cols"]
        img = np.zeros(rows * cols, dtype=np.uint8)
        if not rec["flushed"]:
            img[list(rec["refresh_set"])] = MASK_EDGE_RECOMPUTE
            img[list(rec["reuse_set"])] = MASK_REUSED
        p = out_dir / f"step_{rec['step']:05d}.pgm"
        write_pgm(p, img.reshape(rows, cols))
        paths.append(p)
    return paths

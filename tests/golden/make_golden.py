"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

It imports the reference's own ``freqcache`` package from
/root/reference/pkg/src and records its decisions on the recipes of
``cases.py`` and on the frozen synthetic generator's BASELINE config 1 / 2
sequences.  RGB frames are reduced to gray with the reference's own
``frameio.LUMA_WEIGHTS`` (the same left-to-right expression as
``read_netpbm``), and config 2's "flush on shift > 1 patch" rule is applied
on top of the reference decision exactly as described in DESIGN.md.
Outputs: ``golden_small.json``, ``golden_c1.json``, ``golden_c2.json``,
``golden_step.json`` next to this script.
"""

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

import freqcache as ref  # noqa: E402
from freqcache.frameio import LUMA_WEIGHTS  # noqa: E402

from cases import C1, C2, compare_cases, fhash, frameio_cases, small_cases  # noqa: E402
from freqcache.compare import compare_domains as ref_compare  # noqa: E402
from freqcache.compare import _patch_amplitudes, _position_cosines, _token_stack, _raw_pixels  # noqa: E402
from paper_2604_24391_b200.synth import stream_frames  # noqa: E402


def ref_gray(rgb):
    rgb = rgb.astype(np.float64)
    return LUMA_WEIGHTS[0] * rgb[..., 0] + LUMA_WEIGHTS[1] * rgb[..., 1] + LUMA_WEIGHTS[2] * rgb[..., 2]


def record(d):
    return {
        "step": d.step, "flushed": d.flushed, "sim_freq": d.sim_freq,
        "displacement": [d.displacement.di, d.displacement.dj, d.displacement.di_patches,
                         d.displacement.dj_patches],
        "entropy": [d.entropy.raw, d.entropy.normalized, d.entropy.bin_count],
        "alpha_t": d.alpha_t, "k_reuse": d.k_reuse, "k_candidate": d.k_candidate,
        "k_final": d.k_final, "reuse_set": list(d.reuse_set), "refresh_set": list(d.refresh_set),
        "rows": d.rows, "cols": d.cols, "diagnostic": d.diagnostic,
    }


def cfg_of(c):
    return ref.CacheConfig(
        tau_mig=c.get("tau_mig", 0.12), edge_lambda=c.get("edge_lambda", 0.25),
        budget=ref.BudgetConfig(c.get("alpha_min", 0.08), c.get("alpha_max", 0.5)),
        patch_size=c["patch_size"])


def shift_rule(d, k):
    """Config 2's opt-in rule on a reference decision (flush, no diagnostic)."""
    if d.diagnostic is None and not d.flushed and max(abs(d.displacement.di_patches),
                                                       abs(d.displacement.dj_patches)) > k:
        rec = record(d)
        rec.update(flushed=True, k_candidate=0, k_final=0, reuse_set=[])
        return rec
    return record(d)


def main():
    small = []
    for name, prev, curr, c in small_cases():
        d = ref.decide(prev, curr, cfg_of(c))
        small.append({"name": name, "cfg": c, "prev": fhash(prev), "curr": fhash(curr), "decision": record(d)})
    (HERE / "golden_small.json").write_text(json.dumps(small, indent=0))

    fr = stream_frames(C1["seed"], C1["stream"], C1["steps"], C1["size"], C1["size"])
    cfg = ref.CacheConfig(patch_size=C1["patch"], budget=ref.BudgetConfig(*C1["alpha"]))
    gray = [ref_gray(f) for f in fr]
    c1 = {"recipe": C1, "frames": [fhash(f) for f in fr],
          "decisions": [record(ref.decide(gray[t - 1], gray[t], cfg, step=t)) for t in range(1, len(fr))]}
    (HERE / "golden_c1.json").write_text(json.dumps(c1))

    cfg = ref.CacheConfig(patch_size=C2["patch"])
    c2 = {"recipe": C2, "streams": []}
    for s in range(C2["streams"]):
        fr = stream_frames(C2["seed"], s, C2["steps"], C2["size"], C2["size"])
        gray = [ref_gray(f) for f in fr]
        c2["streams"].append({
            "frames": [fhash(f) for f in fr],
            "decisions": [shift_rule(ref.decide(gray[t - 1], gray[t], cfg, step=t), C2["refresh_shift"])
                          for t in range(1, len(fr))]})
    (HERE / "golden_c2.json").write_text(json.dumps(c2))

    # reference step(): deterministic token_fn, displacement-mapped sourcing
    rng = np.random.default_rng(77)
    frames = [rng.random((64, 64))]
    for _ in range(5):
        frames.append(np.roll(frames[-1], (int(rng.integers(-9, 10)), int(rng.integers(-9, 10))), axis=(0, 1)))
    cfgs = ref.CacheConfig(patch_size=8, budget=ref.BudgetConfig(0.6, 0.6))
    cache = ref.populate_cache(frames[0], 8, ref.default_token_fn)
    steps = []
    for t in range(1, len(frames)):
        d = ref.decide(frames[t - 1], frames[t], cfgs, step=t)
        cache, rep = ref.step(cache, d, frames[t], ref.default_token_fn)
        steps.append({"decision": record(d), "tokens": fhash(cache.tokens), "ages": cache.ages.ravel().tolist(),
                      "n_reused": rep.n_reused, "latency": rep.latency_model_ms})
    seq = ref.run_sequence([rng.random((64, 64)) for _ in range(8)], ref.CacheConfig(patch_size=8))
    (HERE / "golden_step.json").write_text(json.dumps({
        "frames": [fhash(f) for f in frames], "steps": steps,
        "sequence_seed": 77, "sequence_mean_reuse": seq.mean_reuse_ratio, "sequence_speedup": seq.speedup}))
    # compare_domains reports (compare.py:55-114) + the BASELINE-geometry
    # per-patch cosines of one RGB pair (gray via the reference luma weights)
    cmp = []
    for name, frs, c, labels in compare_cases():
        rep = ref_compare(frs, cfg_of(c), edge_labels=labels)
        cmp.append({"name": name, "cfg": c, "frames": [fhash(f) for f in frs], "report": rep})
    fr = stream_frames(C2["seed"], 0, 2, C2["size"], C2["size"])
    g0, g1 = ref_gray(fr[0]), ref_gray(fr[1])
    grid = ref.PatchGrid(g0, C2["patch"])
    vis = _position_cosines(_token_stack(grid, g0, _raw_pixels), _token_stack(grid, g1, _raw_pixels))
    nf = _position_cosines(_patch_amplitudes(grid, g0), _patch_amplitudes(grid, g1))
    (HERE / "golden_compare.json").write_text(json.dumps({
        "cases": cmp, "pair": {"recipe": C2, "frames": [fhash(f) for f in fr],
                               "visual": vis.tolist(), "naive_freq": nf.tolist()}}))
    # frame readers (frameio.py:29-175): outputs or (message, offset)
    import tempfile
    from freqcache.frameio import load_frames
    fio = []
    with tempfile.TemporaryDirectory() as td:
        for name, suffix, data in frameio_cases():
            p = Path(td) / f"{name}{suffix}"
            p.write_bytes(data)
            try:
                frs = load_frames(p)
                fio.append({"name": name, "frames": [fhash(f) for f in frs], "shape": list(frs[0].shape)})
            except Exception as e:  # noqa: BLE001
                fio.append({"name": name, "error": type(e).__name__,
                            "message": str(e).replace(str(p), "<path>"), "offset": getattr(e, "offset", None)})
    (HERE / "golden_frameio.json").write_text(json.dumps(fio, indent=0))
    print("wrote fixtures:", [p.name for p in HERE.glob("golden_*.json")])


if __name__ == "__main__":
    main()

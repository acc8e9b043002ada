"""bench.py contract: the reference arm (CPU) and the GPU arm (``-m gpu``, a
small size) each print one JSON line with the keys the driver reads."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-streams", "2", "--size", "224"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--cpu-streams", "2", "--size", "224"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_world_size_mismatch_is_refused():
    env = dict(os.environ, RANK="0", WORLD_SIZE="4", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2 and "refusing" in r.stderr


@pytest.mark.parametrize("gpus,weak", [(8, False), (2, False), (4, True)])
def test_gpus_flag_launches_ranks(gpus, weak):
    """``bench.py --gpus N`` without torchrun re-launches itself with N ranks
    (the launch path the driver's scaling run uses), here over gloo with
    FC_BENCH_PLUMBING=1: config 5 read literally shards 512 streams into
    512 / N contiguous blocks; --weak keeps 512 per rank; the max-over-ranks
    time and the counter all-reduce reach rank 0, which alone prints."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["FC_BENCH_PLUMBING"] = "1"
    args = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--steps", "3"]
    if weak:
        args.append("--weak")
    r = subprocess.run(args, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["ms_max"] == float(gpus)          # rank r reports 1 + r ms
    total = 512 * gpus if weak else 512
    assert d["streams_total"] == total and sum(d["streams_per_rank"]) == total
    assert d["streams_per_rank"] == [total // gpus] * gpus
    assert [s[0] for s in d["spans"]] == [r * total // gpus for r in range(gpus)]
    assert d["frames"] == total * 3
    assert d["scaling"] == ("weak" if weak else "strong")
    # the weak-scaling leg reported beside the headline: --streams per rank
    assert d["weak_scaling"]["ms_max"] == float(gpus + 1)
    assert d["weak_scaling"]["streams_total"] == 512 * gpus
    assert d["weak_scaling"]["span0"] == [0, 512]


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """The GPU arm's line at a small size: every key the driver and the judge
    read, with self-consistent values."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--streams", "16", "--steps", "4",
                        "--warmup", "3", "--ring", "4", "--cpu-streams", "2", "--cpu-steps", "1",
                        "--e2e-steps", "2", "--sustained-s", "0.2"], capture_output=True, text=True, timeout=900,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["value"] > 0
    assert abs(d["value"] - 16 / (d["ms_per_step"] / 1e3)) / d["value"] < 1e-6
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 16 * 448 * 448 * 3 * 4 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert d["e2e_u8"]["h2d_bytes_per_step"] == 16 * 448 * 448 * 3
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert d["sustained"]["value"] > 0 and d["sustained"]["seconds"] >= 0.16
    assert "sm_mhz" in d["sustained"]["clocks"]
    dc = d["decisions"]
    assert dc["frames"] == 16 * 4 and 0.0 <= dc["reuse_ratio"] <= 1.0 and 0.0 <= dc["flush_rate"] <= 1.0
    assert d["config"]["graph"] is True
    assert d["weak_scaling"]["value"] == d["value"] and d["weak_scaling"]["streams_per_gpu"] == 16


@pytest.mark.gpu
def test_gpu_two_ranks_one_device():
    """The real multi-rank kernel path (not its plumbing stub): 2 ranks over
    gloo sharing cuda:0 (FC_BENCH_DEVICE), strong headline over 16 streams
    in total plus the weak leg at 16 per rank.  Not a scaling measurement."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(FC_BENCH_DEVICE="0", FC_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--streams", "16", "--steps", "4", "--warmup", "3", "--ring", "4",
                        "--e2e-steps", "2", "--sustained-s", "0"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["streams_per_gpu"] == 8
    assert d["decisions"]["frames"] == 16 * 4                 # counters all-reduced over both ranks
    w = d["weak_scaling"]
    assert w["streams_total"] == 32 and w["streams_per_gpu"] == 16 and w["value"] > 0
    assert abs(w["value"] - 32 / (w["ms_per_step"] / 1e3)) / w["value"] < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("graph_steps,no_graph,boost,no_pipeline", [
    (1, False, "0", False), (2, False, "0", False), (1, True, "0", False), (1, False, "296", False),
    (1, True, "148", False), (1, False, "0", True)])
def test_gpu_bench_pipeline_matches_serial(cuda, monkeypatch, graph_steps, no_graph, boost, no_pipeline):
    """The benchmark's own timed path — bench.Pipeline: front of t + 1 beside
    back of t beside the in-place splice of t - 1 on three streams, replayed
    from per-ring-phase CUDA graphs (or chunks of graph_steps steps without
    per-step joins, or eager) — leaves every stream's token cache, ages and
    last decision bit-identical to plain select-then-splice per step: no
    race between the branches, slots or ping-pong buffers — also with extra
    copier CTAs joining each splice from the back's stream (the boost)."""
    import argparse
    import torch
    import bench
    import paper_2604_24391_b200 as fc
    S, R, D = 24, 4, 64
    a = argparse.Namespace(size=448, patch=14, dim=D, no_pipeline=no_pipeline, no_graph=no_graph,
                           graph_steps=graph_steps, refresh_shift=1)
    dev = torch.device("cuda", 0)
    monkeypatch.setenv("FC_BENCH_SPLICE_BOOST", boost)
    pl = bench.Pipeline(a, dev, S, 0, 0, R)
    torch.cuda.synchronize()
    cache0, ages0 = pl.spl.cache[0].clone(), pl.spl.ages[0].clone()   # no splice has run yet
    pl.advance(2 * R + 1)
    t_last = pl.t_next - 1
    pl.spl.step(pl.outs[t_last & 1].src_map, pl.fresh)          # the pending splice of the last step
    torch.cuda.synchronize()
    tok, age = pl.spl.current()

    eng = fc.FreqCacheEngine(S, 448, 448, 14, fmt="rgb", device=dev)
    N = eng.n_tokens
    cache = torch.zeros((2, S, N, D), dtype=torch.bfloat16, device=dev)
    ages = torch.zeros((2, S, N), dtype=torch.int64, device=dev)
    cache[0], ages[0] = cache0, ages0
    ref = fc.SpliceState(cache, ages)
    for t in range(t_last + 1):
        out = eng.select(pl.frames[t % R], pl.cfg, refresh_shift=1)
        ref.step(out.src_map, pl.fresh)
    torch.cuda.synchronize()
    rtok, rage = ref.current()
    last = pl.outs[t_last & 1]
    for name in ("results", "src_map", "reuse_idx", "recompute_idx", "refresh_mask", "energy"):
        assert torch.equal(getattr(last, name), getattr(out, name)), name
    assert torch.equal(tok.view(torch.int16), rtok.view(torch.int16))
    assert torch.equal(age, rage)
    # the run exercised the splice: recomputed rows replaced, reused rows aged,
    # and some streams shifted (ping-pong buffers)
    moved = (tok.view(torch.int16) != cache0.view(torch.int16)).any(-1).float().mean().item()
    assert moved > 0.2 and int(age.max()) >= 2
    assert bool(pl.spl.slot.any()) and not bool(pl.spl.slot.all())
    pl.spl.check()

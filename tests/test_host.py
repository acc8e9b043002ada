"""CPU tests: C-ABI library exports, host-side API logic, multi-rank plumbing."""

import ctypes
import math
import os
import re
import socket
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2604_24391_b200.build import build
    build()
    from paper_2604_24391_b200 import _native
    return _native.load()


def test_library_exports_every_header_symbol(lib):
    hdr = (ROOT / "include" / "freqcache_b200.h").read_text()
    decl = set(re.findall(r"\b(fc_[a-z0-9_]+)\s*\(", hdr))
    assert decl, "no declarations parsed"
    from paper_2604_24391_b200 import _native
    assert decl == set(_native.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    assert lib.fc_abi_version() == 2
    assert lib.fc_strerror(5).decode() == "normalized entropy must lie in [0, 1]"


def test_result_struct_layout():
    from paper_2604_24391_b200 import _native
    assert _native.RESULT_DTYPE.itemsize == 136
    assert ctypes.sizeof(_native.Config) == 40
    assert ctypes.sizeof(_native.Geometry) == 20


def test_plan_rejects_bad_geometry_without_device(lib):
    from paper_2604_24391_b200 import _native
    plan = ctypes.c_void_p()
    for geom in [(1, 30, 30, 8, 0), (1, 32, 32, 1, 0), (0, 32, 32, 8, 0), (1, 32, 32, 8, 7)]:
        rc = lib.fc_plan_create(ctypes.byref(_native.Geometry(*geom)), ctypes.byref(plan))
        assert rc == _native.FC_EINVAL
    rc = lib.fc_plan_create(ctypes.byref(_native.Geometry(1, 4096, 4096, 16, 0)), ctypes.byref(plan))
    assert rc == _native.FC_EUNSUPPORTED


def test_plan_geometry_validation_property(lib):
    """fc_plan_create over random geometries: every invalid one (frame.py:31-37
    rules, bad format) is refused with FC_EINVAL, sizes beyond the kernel
    envelope with FC_EUNSUPPORTED, before any device call; valid ones are never
    refused as invalid (without a device they stop at FC_ECUDA)."""
    from hypothesis import given, settings, strategies as st
    from paper_2604_24391_b200 import _native

    @settings(max_examples=300, deadline=None, derandomize=True)
    @given(st.integers(-2, 6), st.integers(-3, 2000), st.integers(-3, 2000), st.integers(-1, 70),
           st.integers(-2, 7))
    def prop(batch, h, w, p, fmt):
        plan = ctypes.c_void_p()
        rc = lib.fc_plan_create(ctypes.byref(_native.Geometry(batch, h, w, p, fmt)), ctypes.byref(plan))
        invalid = (batch < 1 or h < 1 or w < 1 or p < 2 or h % p or w % p
                   or not (_native.FC_FMT_RGB_F32 <= fmt <= _native.FC_FMT_RGB_U8))
        if invalid:
            assert rc == _native.FC_EINVAL
        elif h > 1536 or w > 1536:
            assert rc == _native.FC_EUNSUPPORTED
        else:
            assert rc in (_native.FC_OK, _native.FC_EUNSUPPORTED, _native.FC_ECUDA)
        if rc == _native.FC_OK:
            lib.fc_plan_destroy(plan)
        else:
            assert not plan.value

    prop()


def test_splice_rejects_bad_arguments_without_device(lib):
    # argument checks return before any device call (fc_abi.cu fc_splice / fc_splice_inplace)
    from paper_2604_24391_b200 import _native
    p = ctypes.c_void_p(4096)   # never dereferenced: every call below is refused first
    big = 1 << 16
    assert lib.fc_splice(big, big, 32, p, p, p, p, 0, 0, p, p, None, None) == _native.FC_EINVAL
    assert lib.fc_splice(1, 4, 32, p, p, p, p, 7, 0, p, p, None, None) == _native.FC_EINVAL
    assert lib.fc_splice(1, 4, 32, p, p, p, p, 1, 0, p, p, None, None) == _native.FC_EINVAL   # compact, no rows
    assert lib.fc_splice_inplace(big, big, 32, p, p, p, p, p, p, p, p, 0, 0, p, None, None) == _native.FC_EINVAL
    assert lib.fc_splice_inplace(1, 4, 24, p, p, p, p, p, p, p, p, 0, 0, p, None, None) == _native.FC_EINVAL
    assert lib.fc_splice_inplace(1, 4, 32, p, p, p, p, p, p, p, p, 1, 0, p, None, None) == _native.FC_EINVAL
    assert lib.fc_splice_inplace(1, 4, 32, p, ctypes.c_void_p(4100), p, p, p, p, p, p, 0, 0, p,
                                 None, None) == _native.FC_EINVAL   # misaligned cache


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    import paper_2604_24391_b200 as fc
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fc.decide(np.random.rand(32, 32), np.random.rand(32, 32), fc.CacheConfig(patch_size=8))


def test_config_validation():
    import paper_2604_24391_b200 as fc
    with pytest.raises(ValueError):
        fc.CacheConfig(tau_mig=1.5)
    with pytest.raises(ValueError):
        fc.CacheConfig(edge_lambda=math.inf)
    with pytest.raises(ValueError):
        fc.CacheConfig(patch_size=1)
    with pytest.raises(ValueError):
        fc.BudgetConfig(0.6, 0.5)


def test_scalar_stage_helpers():
    import paper_2604_24391_b200 as fc
    assert fc.reuse_budget(0.0, fc.BudgetConfig(), 196) == (0.5, 98)
    assert fc.reuse_budget(1.0, fc.BudgetConfig(), 196)[1] == 45
    with pytest.raises(ValueError):
        fc.reuse_budget(1.0000000000000002, fc.BudgetConfig(), 196)
    assert fc.migration_gate(0.12, 0.12) is fc.GateAction.PROCEED
    assert fc.migration_gate(0.0, 0.12) is fc.GateAction.FLUSH
    assert [fc.cutoff_index(p) for p in (2, 4, 8, 16)] == [1, 1, 2, 4]
    assert fc.highpass_filter(8)[:2, :2].sum() == 0 and fc.highpass_filter(8).sum() == 60
    grid = fc.PatchGrid(np.ones((16, 16)), 4)
    assert fc.alignment_mask(fc.Displacement(4, 0, 1, 0), grid).sum() == 12
    assert fc.alignment_mask(fc.Displacement(0, 0, 4, 0), grid).sum() == 0
    for px, exp in [(0, 0), (4, 0), (5, 1), (12, 1), (13, 2), (-4, 0), (-5, -1), (-13, -2)]:
        assert fc.Displacement.from_pixels(px, 0, 8).di_patches == exp


def test_cost_model():
    import paper_2604_24391_b200 as fc
    m = fc.DEFAULT_COST_MODEL
    assert m.latency_ms(196) == pytest.approx(637.0, abs=1e-9)
    assert m.latency_ms(196 * (1 - 0.535)) == pytest.approx(401.0, abs=1e-9)


def test_patch_grid():
    import paper_2604_24391_b200 as fc
    g = fc.PatchGrid(np.arange(64.0).reshape(8, 8), 4)
    assert (g.rows, g.cols, g.n_patches) == (2, 2, 4)
    assert g.position(3) == (1, 1) and g.index(1, 0) == 2
    assert g.blocks().shape == (2, 2, 4, 4)
    with pytest.raises(ValueError):
        fc.PatchGrid(np.ones((10, 8)), 4)
    with pytest.raises(ValueError):
        fc.validate_frame(np.array([[np.nan]]))


def test_shard_covers_streams():
    from paper_2604_24391_b200.dist import shard
    for total in (512, 513, 7):
        for world in (1, 2, 3, 8):
            parts = [shard(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_24391_b200.dist import gather_counters, max_over_ranks, shard, step_counters
    from paper_2604_24391_b200._native import RESULT_DTYPE
    lo, hi = shard(512, world, rank)
    rec = np.zeros(hi - lo, dtype=RESULT_DTYPE)
    rec["rows"], rec["cols"] = 32, 32
    rec["k_final"] = 100 + rank
    rec["flushed"][:3] = 1
    c = gather_counters(step_counters(rec))
    t = max_over_ranks(1.0 + rank)
    q.put((rank, c, t))
    dist.destroy_process_group()


def test_two_rank_gloo_metric_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, c, t in out:
        assert c["frames"] == 512 and c["tokens"] == 512 * 1024
        assert c["reused_tokens"] == 256 * 100 + 256 * 101
        assert c["flushes"] == 6
        assert t == 2.0


def test_psi_status_maps_to_reference_error():
    """FC_EPSI from the select kernel surfaces as budget.py:69-70's ValueError
    (host-side mapping, no device needed)."""
    import numpy as np
    from paper_2604_24391_b200 import _native as nat
    from paper_2604_24391_b200.api import _raise_status
    rec = np.zeros(1, dtype=nat.RESULT_DTYPE)[0]
    rec["status"] = nat.FC_EPSI
    rec["entropy_norm"] = 1.0000000000000002
    with pytest.raises(ValueError, match=r"normalized entropy must lie in \[0, 1\], got 1.0000000000000002"):
        _raise_status(rec)


def test_new_entry_points_refuse_bad_arguments_without_device(lib):
    """Round-2 entry points validate on the host before any device call."""
    import ctypes
    from paper_2604_24391_b200 import _native
    p = ctypes.c_void_p(4096)   # never dereferenced
    E = _native.FC_EINVAL
    assert lib.fc_select_front(None, None, p, p, None, 0, None) == E
    assert lib.fc_select_back(None, None, p, p, None, 0, None) == E
    assert lib.fc_dft2(0, 4, p, 0, 0, p, p, None) == E
    assert lib.fc_dft2(4, 4, None, 0, 0, p, p, None) == E
    assert lib.fc_dft2_workspace_bytes(0, 3) == -1
    assert lib.fc_phase_correlation_spectra(4, 0, p, p, p, p, None) == E
    assert lib.fc_block_dct(1, 65, p, p, None) == E
    assert lib.fc_block_dct(0, 8, None, None, None) == _native.FC_OK      # nothing to do
    assert lib.fc_amplitude_phase(-1, p, p, p, None) == E
    assert lib.fc_gather_patches(-1, 1, 28, 28, 14, p, p, p, None) == E
    assert lib.fc_gather_patches(4, 1, 30, 28, 14, p, p, p, None) == E     # P does not divide H
    assert lib.fc_graph_launch(None, None) == E
    assert lib.fc_graph_capture_end(None, None) == E
    assert lib.fc_plan_launches(None) == -1
    # the split in-place splice: same argument rules as fc_splice_inplace
    args = (2, 16, 64, p, p, p, p, p, p, p, p, _native.FC_FRESH_DENSE, 16, p)
    assert lib.fc_splice_inplace_plan(0, *args[1:], None) == E                  # batch < 1
    assert lib.fc_splice_inplace_plan(2, 16, 60, *args[3:], None) == E          # row bytes not a multiple of 16
    assert lib.fc_splice_inplace_plan(*args[:3], None, *args[4:], None) == E    # no src_map
    assert lib.fc_splice_inplace_copy(*args, p, -1, None) == E                   # negative CTA count
    assert lib.fc_splice_inplace_copy(*args[:11], 7, *args[12:], p, 0, None) == E   # bad fresh layout


def test_header_is_plain_c_and_the_c_example_links(lib, tmp_path):
    """The boundary is a C ABI: the header compiles as strict C99 on its own
    (no C++ or torch types), and examples/select_c.c — the ABI driven from
    plain C through cudart — builds and links against the in-tree library
    (it runs in the GPU suite)."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    src = tmp_path / "h.c"
    src.write_text('#include "freqcache_b200.h"\nint main(void) { fc_geometry g = {1, 16, 16, 8, FC_FMT_GRAY_F32};'
                   ' return g.batch - 1 + (int)sizeof(fc_stream_result) * 0; }\n')
    r = subprocess.run([gcc, "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                        f"-I{ROOT / 'include'}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    cuda_inc = Path("/usr/local/cuda/include/cuda_runtime_api.h")
    if not cuda_inc.exists() or shutil.which("make") is None:
        pytest.skip("no CUDA headers / make")
    r = subprocess.run(["make", "-s", "-C", str(ROOT / "examples"), "select_c"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert (ROOT / "examples" / "select_c").exists()

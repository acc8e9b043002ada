"""pytest plugin: run the reference's own test corpus against the B200 facade.

TEST INFRASTRUCTURE.  Used by ``tests/test_gpu_reference_corpus.py`` as

    PYTHONPATH=tests/refcorpus python -m pytest -p fc_refcorpus_plugin <staged reference tests>

The reference's tests (``pkg/tests``, staged unmodified into
``baseline/_ref/corpus_tests`` by ``scripts/stage_reference.sh``) import the
package ``freqcache``.  This plugin installs a ``freqcache`` module tree
into ``sys.modules`` whose names resolve to this repository's GPU facade
(``paper_2604_24391_b200``): decide / step / run_sequence, the stage
functions, the fp64 transform wrappers, types, frame I/O, records and the
comparison baselines.  Names the tier leaves out of scope come from the
unmodified reference installed in ``baseline/_ref`` (loaded under the
package name ``freqcache_ref``): the scene generator (``scenes``), the
in-package slow twin ``decide_reference`` (the corpus's own oracle), and the
``bench`` / ``cli`` harness modules — whose references to path functions
are rebound to the facade, so their tests drive the GPU path.

Floats are re-toleranced as SURVEY §4 prescribes: the corpus's
``oracles.assert_decision_equivalence`` keeps every discrete field exact and
compares sim / alpha / entropy within 1e-3 (its default was 1e-9, an fp64
transform-path tolerance an fp32 GPU FFT cannot meet).
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref", "freqcache")
FLOAT_TOL = 1e-3

SUBMODULES = ("frame", "errors", "spectral", "migration", "edge_refresh", "budget", "fusion", "frameio", "records",
              "compare", "scenes", "bench", "cli")


def _load_reference():
    """The unmodified reference package under the name ``freqcache_ref``."""
    if "freqcache_ref" in sys.modules:
        return sys.modules["freqcache_ref"]
    spec = importlib.util.spec_from_file_location("freqcache_ref", os.path.join(REF, "__init__.py"),
                                                  submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["freqcache_ref"] = mod
    spec.loader.exec_module(mod)
    for name in SUBMODULES:
        importlib.import_module(f"freqcache_ref.{name}")
    return mod


def _facade_names():
    import paper_2604_24391_b200 as fc
    from paper_2604_24391_b200 import compare as fc_compare
    from paper_2604_24391_b200 import frameio as fc_frameio
    from paper_2604_24391_b200 import records as fc_records
    from paper_2604_24391_b200 import spectral as fc_spectral
    from paper_2604_24391_b200 import stages as fc_stages
    names = {k: getattr(fc, k) for k in dir(fc) if not k.startswith("__")}
    for m in (fc_stages, fc_spectral, fc_records, fc_frameio, fc_compare):
        names.update({k: getattr(m, k) for k in dir(m) if not k.startswith("__") and not isinstance(
            getattr(m, k), types.ModuleType)})
    names["export_masks"] = fc_records.export_masks
    return names


def _as_facade_decision(d):
    """A reference CacheDecision as the facade's type, field for field, so
    the corpus's equality checks compare values, not dataclass classes."""
    import paper_2604_24391_b200 as fc
    return fc.CacheDecision(
        step=d.step, flushed=d.flushed, sim_freq=d.sim_freq,
        displacement=fc.Displacement(d.displacement.di, d.displacement.dj, d.displacement.di_patches,
                                     d.displacement.dj_patches),
        entropy=fc.EntropyReading(d.entropy.raw, d.entropy.normalized, d.entropy.bin_count),
        alpha_t=d.alpha_t, k_reuse=d.k_reuse, k_candidate=d.k_candidate, k_final=d.k_final,
        reuse_set=tuple(d.reuse_set), recompute_set=tuple(d.recompute_set), rows=d.rows, cols=d.cols,
        refresh_set=tuple(d.refresh_set), diagnostic=d.diagnostic, timings_us=dict(d.timings_us))


def install():
    ref = _load_reference()
    facade = _facade_names()
    ref_twin = ref.decide_reference

    def decide_reference(*args, **kwargs):
        return _as_facade_decision(ref_twin(*args, **kwargs))

    decide_reference.__doc__ = "The reference's slow twin (fusion.py:265-398), result as facade types."
    top = types.ModuleType("freqcache")
    top.__path__ = []          # a package, so `freqcache.x` submodules resolve
    top.__file__ = __file__
    sys.modules["freqcache"] = top
    for name in SUBMODULES:
        refmod = sys.modules[f"freqcache_ref.{name}"]
        sub = types.ModuleType(f"freqcache.{name}")
        if name in ("scenes",):
            src = dict(vars(refmod))                      # out of scope: the reference's generator
        elif name in ("bench", "cli"):
            # the reference's harness code, with the path functions it calls
            # rebound to the facade
            src = dict(vars(refmod))
            for k in list(vars(refmod)):
                if k in facade and not k.startswith("_") and k not in ("SCENE_KINDS", "SceneSpec",
                                                                        "generate_scene", "Scene"):
                    setattr(refmod, k, facade[k])
                    src[k] = facade[k]
        else:
            # every public name of the reference module, from the facade;
            # the reference's slow twin (decide_reference) stays the
            # reference's — it is the corpus's own oracle
            src = {}
            for k, v in vars(refmod).items():
                if k.startswith("__"):
                    continue
                if k == "decide_reference":
                    src[k] = decide_reference
                elif k.startswith("_"):
                    src[k] = v
                elif k in facade:
                    src[k] = facade[k]
                else:
                    src[k] = v
        for k, v in src.items():
            if not k.startswith("__"):
                setattr(sub, k, v)
        sys.modules[f"freqcache.{name}"] = sub
        setattr(top, name, sub)
    for k, v in vars(ref).items():
        if k.startswith("__") and k != "__version__":
            continue
        if isinstance(v, types.ModuleType):
            continue
        setattr(top, k, facade.get(k, v) if k != "decide_reference" else decide_reference)
    top.__all__ = list(getattr(ref, "__all__", []))


def pytest_configure(config):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    install()
    # oracles.py sits beside the corpus tests: re-tolerance its decision
    # comparison (discrete fields stay exact, floats within FLOAT_TOL)
    for arg in config.args:
        d = arg if os.path.isdir(arg) else os.path.dirname(arg)
        if os.path.exists(os.path.join(d, "oracles.py")):
            if d not in sys.path:
                sys.path.insert(0, d)
            mod = importlib.import_module("oracles")
            mod.assert_decision_equivalence.__defaults__ = (FLOAT_TOL,)
            break

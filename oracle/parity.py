"""Margin-aware parity checker — TEST INFRASTRUCTURE ONLY.

Compares a device decision (anything with CacheDecision's fields) with an
``OracleDecision``.  Discrete outputs must be bit-exact except where the
oracle's own margin to the decision threshold is <= ``REL`` (1e-4 relative):

* refresh mask, per token: |E - thr| / |thr|;
* top-K membership/order, per token: distance to the K boundary, with an
  absolute floor of 1e-6 * mean(E) so fp64 rounding-noise ties count as ties;
* displacement, per step: (r1 - r2) / r1 of the correlation peak (a flip
  exempts everything that depends on the alignment);
* K = floor(alpha N), per step: distance of alpha N to an integer;
* the gate, per step: |sim - tau| / tau;
* psi within 1e-6 of 1 (fp32 cannot reproduce an fp64 1-ulp overshoot).

Floats (sim, psi, alpha, energies) must agree within ``FTOL`` (1e-3) relative;
energies additionally within the fp64 rounding floor of a patch energy,
64 u P^2 s^2 (u = 2^-53, s = the frame's largest gray value, 1 for [0, 1]
frames): both sides compute E as a difference of sums over P^2 squares, so a
constant patch is ~1e-31 in the reference (DCT rounding) and ~1e-15 in the
Parseval form, both numerically zero.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .freqcache_oracle import OracleConfig, OracleDecision, decision_margins

REL = 1e-4
FTOL = 1e-3


@dataclass
class ParityReport:
    ok: bool = True
    errors: list = field(default_factory=list)
    exemptions: dict = field(default_factory=dict)

    def fail(self, msg):
        self.ok = False
        self.errors.append(msg)

    def exempt(self, kind, n=1):
        self.exemptions[kind] = self.exemptions.get(kind, 0) + n


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def compare(dev, ora: OracleDecision, cfg: OracleConfig, energies=None, rep=None, frame_scale=1.0):
    """Check one step.  ``energies``: device per-token energies (optional);
    ``frame_scale``: largest gray value of the frames (energy rounding floor)."""
    rep = rep or ParityReport()
    m = decision_margins(ora, cfg)
    n = ora.rows * ora.cols

    if (dev.rows, dev.cols) != (ora.rows, ora.cols):
        rep.fail("grid shape")
        return rep
    if dev.diagnostic != ora.diagnostic:
        rep.fail(f"diagnostic {dev.diagnostic!r} != {ora.diagnostic!r}")
        return rep

    # ---- floats
    if energies is not None:
        e_ref = ora.energies
        floor = 1e-6 * float(e_ref.mean()) if e_ref.size else 0.0
        floor = max(floor, 64.0 * 2.0 ** -53 * cfg.patch_size ** 2 * float(frame_scale) ** 2)
        err = np.abs(np.asarray(energies, dtype=np.float64) - e_ref)
        bad = err > FTOL * np.abs(e_ref) + floor
        if bad.any():
            q = int(np.flatnonzero(bad)[0])
            rep.fail(f"energy[{q}] {energies[q]!r} vs {e_ref[q]!r}")
    if ora.diagnostic is None and _rel(dev.sim_freq, ora.sim_freq) > FTOL:
        rep.fail(f"sim_freq {dev.sim_freq} vs {ora.sim_freq}")
    psi_d, psi_o = dev.entropy.normalized if hasattr(dev.entropy, "normalized") else dev.entropy[1], ora.entropy[1]
    if abs(psi_d - psi_o) > FTOL * max(abs(psi_o), 1e-12) + 1e-9:
        rep.fail(f"psi {psi_d} vs {psi_o}")
    if _rel(dev.alpha_t, ora.alpha_t) > FTOL and abs(dev.alpha_t - ora.alpha_t) > 1e-12:
        rep.fail(f"alpha {dev.alpha_t} vs {ora.alpha_t}")

    # ---- refresh mask
    fr_d, fr_o = set(dev.refresh_set), set(ora.refresh_set)
    flips = fr_d ^ fr_o
    for q in flips:
        if m["refresh"][q] <= REL:
            rep.exempt("refresh")
        else:
            rep.fail(f"refresh flip at {q} (margin {m['refresh'][q]:.3g})")

    # ---- budget
    k_ok = dev.k_reuse == ora.k_reuse
    if not k_ok:
        if m["k"] <= REL and abs(dev.k_reuse - ora.k_reuse) <= 1:
            rep.exempt("k_reuse")
        else:
            rep.fail(f"k_reuse {dev.k_reuse} vs {ora.k_reuse}")

    # ---- gate / flush
    if dev.flushed != ora.flushed:
        if m["gate"] <= REL or m["disp"] <= REL:
            rep.exempt("flush")
            return rep
        rep.fail(f"flushed {dev.flushed} vs {ora.flushed}")
        return rep

    # ---- displacement
    dd = tuple(dev.displacement) if not hasattr(dev.displacement, "di") else (
        dev.displacement.di, dev.displacement.dj, dev.displacement.di_patches, dev.displacement.dj_patches)
    if dd != tuple(ora.displacement):
        if m["disp"] <= REL:
            rep.exempt("displacement")
            return rep
        rep.fail(f"displacement {dd} vs {ora.displacement}")
        return rep

    if ora.flushed:
        if dev.k_final or dev.k_candidate or dev.reuse_set:
            rep.fail("flushed step reuses tokens")
        return rep

    # ---- candidates / top-K
    k_cand_slack = len([q for q in flips if ora.align is None or ora.align[q]])
    if abs(dev.k_candidate - ora.k_candidate) > k_cand_slack:
        rep.fail(f"k_candidate {dev.k_candidate} vs {ora.k_candidate}")
    ru_d, ru_o = set(dev.reuse_set), set(ora.reuse_set)
    diff = ru_d ^ ru_o
    if diff:
        ambiguous = {q for q in diff if m["topk"][q] <= REL or q in flips}
        rest = diff - ambiguous
        if rest and (flips or not k_ok):
            # a flipped candidate or a +-1 budget moves the K boundary by one
            e = ora.energies
            cand = [q for q in range(n) if ora.align[q] and q not in fr_o]
            ranked = sorted(cand, key=lambda q: (e[q], q))
            w = len(flips) + (0 if k_ok else 1)
            k = ora.k_final
            window = set(ranked[max(0, k - w - 1): k + w + 1])
            ambiguous |= rest & window
            rest -= window
        if rest:
            rep.fail(f"reuse set differs at {sorted(rest)[:8]}")
        else:
            rep.exempt("reuse_membership", len(diff))
    # order of the common tokens
    common = ru_d & ru_o
    seq_d = [q for q in dev.reuse_set if q in common]
    seq_o = [q for q in ora.reuse_set if q in common]
    if seq_d != seq_o:
        e = ora.energies
        floor = m["energy_floor"]
        pos = {q: i for i, q in enumerate(seq_o)}
        for a, b in zip(seq_d, seq_d[1:]):
            if pos[a] > pos[b]:
                gap = abs(e[a] - e[b])
                if gap <= REL * max(e[a], e[b]) + floor:
                    rep.exempt("order")
                else:
                    rep.fail(f"reuse order {a} before {b} (E {e[a]!r} vs {e[b]!r})")
                    break
    if sorted(dev.recompute_set) != sorted(set(range(n)) - ru_d) or list(dev.recompute_set) != sorted(dev.recompute_set):
        rep.fail("recompute set is not the row-major complement")
    return rep

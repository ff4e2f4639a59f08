"""Parity comparator: CUDA path vs fp64 oracle (DESIGN.md s.4).

Tolerances (BASELINE.json north_star + the arithmetic):
  * subray prim ids bit-exact; where the oracle's candidate set (every
    triangle within 1e-6 m of the nearest, exported as ids) has more than one
    member, a DIFFERENT id is accepted only if it lies in that set -- and that
    subray is then "tie-taken": its amplitude is not compared and its pulse is
    exempt from the waveform / return checks (the neighbour may have another
    normal or reflectance);
  * ranges |dr| <= 1e-6 r + 1e-5 m;
  * amplitudes / intensities / waveform bins within 1e-4 relative (zero must
    be exactly zero);
  * voxel transmission decisions exact, except where |u - exp(-sigma L)| <=
    1e-12 (exempt subray);
  * k_s exact except where the oracle's k-margin <= 1e-9 (exempt subray);
  * per pulse: k0 exact; n_returns exact unless a peak decision's margin is
    <= DECISION_EPS = 2.5e-7 (the GPU bins fp32-rounded amplitudes: every bin
    within 6e-8 relative, so a comparison flips only within 1.2e-7); return
    ranges within 1e-12 relative, intensities within 1e-4; return prim ids in
    the oracle's attribution set (the distinct prims whose contribution is
    within DECISION_EPS of the largest; usually one);
  * exemption budget: exempt pulses <= 1e-4 of the pulses compared
    (Report.budget_ok), by reason in Report.exempt_pulses.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

C = 299792458.0
MISS = 0xFFFFFFFF
DECISION_EPS = 2.5e-7
EXEMPT_BUDGET = 1e-4


@dataclass
class Report:
    pulses: int = 0
    subrays: int = 0
    exempt_subrays: dict = field(default_factory=dict)
    exempt_pulses: dict = field(default_factory=dict)
    checked: dict = field(default_factory=dict)
    mismatches: list = field(default_factory=list)
    max_rel: dict = field(default_factory=dict)

    def bump(self, d, k, n=1):
        d[k] = d.get(k, 0) + int(n)

    def fail(self, what, idx, detail=""):
        if len(self.mismatches) < 50:
            self.mismatches.append(f"{what} @ {idx} {detail}")
        else:
            self.mismatches.append("...")

    def rel(self, k, v):
        self.max_rel[k] = max(self.max_rel.get(k, 0.0), float(v))

    def ok(self):
        return not self.mismatches

    def n_exempt_pulses(self):
        return sum(self.exempt_pulses.values())

    def budget_ok(self, frac: float = EXEMPT_BUDGET):
        """Exempt pulses within the C-4 budget (<= frac of those compared)."""
        return self.n_exempt_pulses() <= frac * self.pulses

    def summary(self):
        return (f"pulses={self.pulses} subrays={self.subrays} exempt_subrays={self.exempt_subrays}"
                f" exempt_pulses={self.exempt_pulses} checked={self.checked}"
                f" max_rel={self.max_rel} mismatches={len(self.mismatches)}: {self.mismatches[:10]}")

    def table_row(self, name: str) -> str:
        ex = ", ".join(f"{k} {v}" for k, v in sorted(self.exempt_pulses.items()) if v) or "none"
        exs = ", ".join(f"{k} {v}" for k, v in sorted(self.exempt_subrays.items()) if v) or "none"
        mr = ", ".join(f"{k} {v:.2e}" for k, v in sorted(self.max_rel.items()))
        return (f"| {name} | {self.pulses} | {self.subrays} | {exs} | {ex} | "
                f"{self.n_exempt_pulses() / max(1, self.pulses):.1e} | {len(self.mismatches)} | {mr} |")


def record(name: str, rep: Report) -> None:
    """Append the report's row to the exemption table named by
    $HELIOS_PARITY_TABLE (profiles/<round>_parity_exemptions.md), if set."""
    import os
    path = os.environ.get("HELIOS_PARITY_TABLE")
    if not path:
        return
    new = not os.path.exists(path)
    with open(path, "a") as f:
        if new:
            f.write("| case | pulses | subrays | exempt subrays | exempt pulses | exempt frac | "
                    "mismatches | max rel |\n|---|---|---|---|---|---|---|---|\n")
        f.write(rep.table_row(name) + "\n")


def _in_set(ids: np.ndarray, sets: np.ndarray) -> np.ndarray:
    """ids [...]: is ids[...] one of sets[..., :] (UINT32_MAX-padded)?"""
    return np.any(sets == ids[..., None], axis=-1) & (ids != MISS)


def compare(gpu: dict, orc, n_tris: int, bin_width_ns: float, report: Report | None = None,
            check_waveform: bool = True, fit_span_ns: float | None = None) -> Report:
    """gpu: Outputs.numpy() (with subray_hits); orc: oracle.OracleResult on the
    same pulses in the same order."""
    r = report or Report()
    n, N = orc.sub_range.shape
    r.pulses += n
    r.subrays += n * N
    sh = gpu["subray_hits"]
    g_prim = sh["prim_id"].astype(np.int64)
    g_rng = sh["range_m"]
    g_amp = sh["amplitude"].astype(np.float64)
    o_prim = orc.sub_prim.astype(np.int64)
    o_rng = orc.sub_range
    o_amp = orc.sub_amp

    same = g_prim == o_prim
    umarg = orc.sub_umargin <= 1e-12
    kmarg = orc.sub_kmargin <= 1e-9
    multi = orc.sub_ncand > 1
    in_cand = _in_set(sh["prim_id"].astype(np.uint32), orc.sub_cand)
    # a listed candidate other than the oracle's choice: legitimate, exempt
    tie_taken = ~same & multi & in_cand & ~umarg
    # more candidates than the oracle lists and the GPU's id not among them:
    # cannot be verified by id; counted (expected 0) and checked by range
    overflow = ~same & (orc.sub_ncand > orc.sub_cand.shape[-1]) & ~in_cand & ~umarg
    r.bump(r.exempt_subrays, "tie_taken", tie_taken.sum())
    r.bump(r.exempt_subrays, "tie_overflow", overflow.sum())
    r.bump(r.exempt_subrays, "u_margin", umarg.sum())
    r.bump(r.exempt_subrays, "k_margin", kmarg.sum())
    r.bump(r.checked, "tie_subrays_same_id", (same & multi).sum())
    sub_ex = tie_taken | overflow | umarg
    # --- per subray: prim ids
    bad = ~same & ~sub_ex
    for i, s in zip(*np.nonzero(bad)):
        r.fail("subray prim", (i, s), f"gpu={g_prim[i, s]} oracle={o_prim[i, s]} "
                                      f"r_gpu={g_rng[i, s]} r_or={o_rng[i, s]} "
                                      f"cand={orc.sub_cand[i, s][:orc.sub_ncand[i, s]]}")
    # --- ranges (every hit, incl. tie-taken ones: the candidates lie within 1e-6 m)
    both_hit = (g_prim != MISS) & (o_prim != MISS)
    sel = both_hit & ~umarg
    dr = np.abs(g_rng[sel] - o_rng[sel])
    lim = 1e-6 * np.abs(o_rng[sel]) + 1e-5
    if sel.any():
        r.rel("range_abs", dr.max())
        for k in np.nonzero(dr > lim)[0][:10]:
            r.fail("subray range", k, f"{g_rng[sel][k]} vs {o_rng[sel][k]}")
    # --- amplitudes
    sel = both_hit & same & ~umarg
    if sel.any():
        a, b = g_amp[sel], o_amp[sel]
        rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-300)
        rel[(a == 0) & (b == 0)] = 0
        r.rel("amplitude", rel.max())
        for k in np.nonzero(rel > 1e-4)[0][:10]:
            r.fail("subray amplitude", k, f"{a[k]} vs {b[k]}")
    # --- k_s
    sel = both_hit & same & ~umarg & ~kmarg
    g_k = np.floor(2.0 * g_rng[sel] / C / (bin_width_ns * 1e-9)).astype(np.int64)
    if sel.any():
        badk = g_k != orc.sub_k[sel]
        for k in np.nonzero(badk)[0][:10]:
            r.fail("subray k_s", k, f"{g_k[k]} vs {orc.sub_k[sel][k]}")

    # --- per pulse
    p_sub_ex = (sub_ex | kmarg).any(axis=1)
    p_peak_ex = (orc.peak_margin <= DECISION_EPS) & ~p_sub_ex
    r.bump(r.exempt_pulses, "subray", p_sub_ex.sum())
    r.bump(r.exempt_pulses, "peak_margin", p_peak_ex.sum())
    g_k0 = gpu["wf_first_bin"]
    g_nr = gpu["n_returns"].astype(np.int64)
    ret = gpu["returns"]
    for i in range(n):
        if p_sub_ex[i]:
            continue
        if g_k0[i] != orc.k0[i]:
            r.fail("k0", i, f"{g_k0[i]} vs {orc.k0[i]}")
            continue
        if check_waveform and gpu.get("waveform") is not None and orc.waveform is not None:
            gw = gpu["waveform"][i].astype(np.float64)
            ow = orc.waveform[i]
            zero_bad = (ow == 0) != (gw == 0)
            if zero_bad.any():
                r.fail("waveform zero pattern", i, f"{np.nonzero(zero_bad)[0][:5]}")
            nz = ow != 0
            if nz.any():
                rel = np.abs(gw[nz] - ow[nz]) / np.abs(ow[nz])
                r.rel("waveform", rel.max())
                if rel.max() > 1e-4:
                    r.fail("waveform bin", i, f"max rel {rel.max()}")
        if p_peak_ex[i]:
            continue
        if g_nr[i] != orc.n_returns[i]:
            r.fail("n_returns", i, f"{g_nr[i]} vs {orc.n_returns[i]}")
            continue
        m = int(g_nr[i])
        if m == 0:
            continue
        gr = ret[i, :m]
        if not np.array_equal(gr["return_number"], np.arange(1, m + 1)) or np.any(
                gr["n_returns"] != m):
            r.fail("return numbering", i)
        rr = np.abs(gr["range_m"] - orc.ret_range[i, :m]) / np.maximum(
            np.abs(orc.ret_range[i, :m]), 1e-300)
        r.rel("return_range", rr.max())
        if rr.max() > 1e-12:
            r.fail("return range", i, f"{gr['range_m']} vs {orc.ret_range[i, :m]}")
        ri = np.abs(gr["intensity"].astype(np.float64) - orc.ret_intensity[i, :m]) / np.abs(
            orc.ret_intensity[i, :m])
        r.rel("return_intensity", ri.max())
        if ri.max() > 1e-4:
            r.fail("return intensity", i)
        if not np.array_equal(gr["gps_time_s"], orc.ret_time[i, :m]):
            r.fail("return gps time", i)
        # attribution (R13): the GPU's prim must be in the oracle's set
        gp = gr["prim_id"].astype(np.uint32)
        okp = _in_set(gp, orc.ret_cand[i, :m])
        r.bump(r.checked, "returns", m)
        r.bump(r.checked, "returns_attr_tied", int((orc.ret_cand[i, :m, 1] != MISS).sum()))
        r.bump(r.checked, "returns_attr_other_tied_prim",
               int((okp & (gp != orc.ret_prim[i, :m])).sum()))
        if not okp.all():
            r.fail("return prim", i, f"{gp} vs {orc.ret_prim[i, :m]} sets {orc.ret_cand[i, :m]}")
        # echo width (R28): NaN <=> NaN (not requested / not
        # converged), else the same least-squares optimum within 1e-6 relative
        # (both fit in fp64 to a 1e-10 relative step; the GPU's fp32 record adds 6e-8)
        if "echo_width_ns" in gr.dtype.names:
            gw_ = gr["echo_width_ns"].astype(np.float64)
            ow_ = orc.ret_width[i, :m]
            # a width within 1e-3 of the identifiability bound (R28) may
            # land on either side of it: exempt
            fin = np.where(np.isnan(ow_), gw_, ow_)
            edge = (fit_span_ns is not None) & (np.abs(np.abs(fin) - (fit_span_ns or 0))
                                                 <= 1e-3 * (fit_span_ns or 1))
            r.bump(r.checked, "width_bound", int(edge.any()))
            if np.any((np.isnan(gw_) != np.isnan(ow_)) & ~edge):
                r.fail("echo width NaN pattern", i, f"{gw_} vs {ow_}")
            else:
                f = ~np.isnan(ow_)
                f &= ~np.isnan(gw_) & ~edge
                if f.any():
                    rw = np.abs(gw_[f] - ow_[f]) / np.abs(ow_[f])
                    r.rel("echo_width", rw.max())
                    if rw.max() > 1e-6:
                        r.fail("echo width", i, f"{gw_} vs {ow_}")
    return r


def jstar_of(params) -> int:
    """j* = argmax_j p[j] of the binned outgoing pulse (R12), for the invariants."""
    tau = params.pulse_length_ns / 1.75
    taps = int(np.ceil(20.0 * tau / params.bin_width_ns))
    x = (np.arange(taps) + 0.5) * params.bin_width_ns / tau
    return int(np.argmax(x * x * np.exp(-x)))


def gpu_invariants(gpu: dict, max_returns: int, thr: float, params=None) -> list:
    """Properties that hold for every pulse at any size (checked on whole runs)."""
    errs = []
    k0 = gpu["wf_first_bin"]
    nr = gpu["n_returns"].astype(np.int64)
    ret = gpu["returns"]
    wf = gpu.get("waveform")
    if np.any(nr > max_returns):
        errs.append("n_returns > max_returns")
    if np.any(nr[k0 < 0] != 0):
        errs.append("k0 = -1 with returns")
    if wf is not None:
        nohit = k0 < 0
        if np.any(wf[nohit] != 0):
            errs.append("k0 = -1 with a non-zero row")
        if np.any(~wf[~nohit].any(axis=1) & (nr[~nohit] > 0)):
            errs.append("returns from an all-zero row")
    # ranges strictly increasing within a pulse; slots beyond n_returns zeroed
    R = ret.shape[1]
    idx = np.arange(R)[None, :]
    used = idx < nr[:, None]
    rng = ret["range_m"]
    with np.errstate(invalid="ignore"):
        inc = np.diff(np.where(used, rng, np.inf), axis=1)
    if np.any((inc <= 0) & used[:, 1:]):
        errs.append("return ranges not increasing")
    raw = ret.view(np.uint8).reshape(ret.shape[0], R, 32) if ret.dtype.itemsize == 32 else None
    if raw is not None and np.any(raw[~used].any(axis=-1)):
        errs.append("unused return slot not zeroed")
    if wf is not None and params is not None and not getattr(params, "range_noise_sd_m", 0.0):
        # each return's bin (from its range, R12; without ranging noise) is a
        # local maximum >= thr * max of the stored fp32 row (>=: fp32 rounding
        # may equalise neighbours)
        js = jstar_of(params)
        half = 0.5 * C * params.bin_width_ns * 1e-9
        p_idx, r_idx = np.nonzero(used)
        kb = np.rint(rng[p_idx, r_idx] / half - 0.5 - k0[p_idx] + js).astype(np.int64)
        nb = wf.shape[1]
        if np.any((kb < 1) | (kb > nb - 2)):
            errs.append("return bin outside [1, n_bins - 2]")
        else:
            w = wf[p_idx, kb].astype(np.float64)
            wl = wf[p_idx, kb - 1].astype(np.float64)
            wr = wf[p_idx, kb + 1].astype(np.float64)
            M = wf.max(axis=1).astype(np.float64)[p_idx]
            if np.any((w < wl) | (w < wr)):
                errs.append("a return bin is not a local maximum of the stored row")
            if np.any(w < np.float32(thr) * M * (1 - 1e-6)):
                errs.append("a return bin is below the threshold of the stored row")
            if not np.array_equal(ret["intensity"][p_idx, r_idx], wf[p_idx, kb]):
                errs.append("return intensity != stored row at its bin")
    return errs

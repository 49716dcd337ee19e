"""Shared statistics of tools/parity_numbers.py and tools/oracle_noise.py."""
import numpy as np

FLOOR = 1e-12


def hist_stats(h, r):
    h, r = np.asarray(h, dtype=float), np.asarray(r, dtype=float)
    if h.size != r.size:
        return {"hist_len_mismatch": [int(h.size), int(r.size)]}
    rel = np.abs(h - r) / np.maximum(np.abs(r), 1e-300)
    above = np.abs(r) > FLOOR
    return {"hist_rel_max": float(rel.max()) if rel.size else 0.0,
            "hist_rel_max_above_floor": float(rel[above].max()) if above.any() else 0.0,
            "hist_entries": int(r.size), "hist_entries_below_floor": int((~above).sum()),
            "hist_abs_max_below_floor": float(np.abs(h - r)[~above].max()) if (~above).any()
            else 0.0}

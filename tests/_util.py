"""Shared numerics helpers of the parity tests."""
import numpy as np

# north_star: attention outputs within 1e-3 relative in fp32
REL_TOL = 1e-3


def rel_err(got, want) -> float:
    """||got - want||_inf / ||want||_inf -- a true relative bound (no max(1, .)
    floor: attention outputs over ~26K N(0,1) value rows are ~1e-2 in size)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = float(np.abs(want).max()) if want.size else 0.0
    num = float(np.abs(got - want).max()) if want.size else 0.0
    return num / den if den > 0 else num


def selected_rows(bits_row, s_mid):
    """Ascending middle rows set in one head's selection words (bit r of word w = row 32w + r)."""
    bits_row = np.ascontiguousarray(bits_row).view(np.uint32)
    return np.flatnonzero(np.unpackbits(bits_row.view(np.uint8), bitorder="little")[:s_mid])

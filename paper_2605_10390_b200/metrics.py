"""Host-side metric arithmetic used by bench.py (no GPU work here).

unit_throughput   T_unit = n / (t * n_c)            PAPER.md:417 §IV.E
bandwidth_eff     b_eff = T_actual / B_DRAM          PAPER.md:432-436 Eq. 1 (useful / total bytes)
roofline_frac     achieved bytes/s / peak bytes/s    BASELINE.json metric
minimal_bytes     read p/8 + write p/8 per key       SURVEY.md §8(d); "p/8 bytes per key"
"""
from __future__ import annotations


def unit_throughput(n: float, t_s: float, n_c: int) -> float:
    if t_s <= 0 or n_c < 1:
        raise ValueError("t must be > 0 and n_c >= 1")
    return n / (t_s * n_c)


def bandwidth_efficiency(useful_bytes: float, total_bytes: float) -> float:
    if total_bytes <= 0:
        raise ValueError("total traffic must be > 0")
    return useful_bytes / total_bytes


def minimal_bytes_keys(n: int, key_bytes: int) -> int:
    """Read every key once and write it once: the floor of any out-of-place sort."""
    return 2 * n * key_bytes


def minimal_bytes_pairs(n: int, key_bytes: int, val_bytes: int) -> int:
    return 2 * n * (key_bytes + val_bytes)


def roofline_frac(bytes_moved: float, t_s: float, peak_gbs: float) -> float:
    return (bytes_moved / t_s) / (peak_gbs * 1e9)

"""ORACLE — TEST INFRASTRUCTURE ONLY: the paper's roofline model (§3).

Eq. 1  P = I * b_S                                  PAPER.md:553-556 (eq:upper_performance)
Eq. 2  I_SpMV(α) = 2 / (8 + 4 + 8α + 20/NNZR)       PAPER.md:585-589 (eq:SpMV_intensity)
Eq. 3  I_SymmSpMV(α) = 4 / (8 + 4 + 24α + 4/SymmNNZR) PAPER.md:746-750 (eq:SymmSpMV_intensity)
Eq. 4  SymmNNZR = (NNZR - 1)/2 + 1                  PAPER.md:751-752 (eq:NNZR_symm)
α_opt = 1/NNZR (SpMV), 1/SymmNNZR (SymmSpMV)
"""
from __future__ import annotations


def symm_nnzr(nnzr: float) -> float:
    return (nnzr - 1.0) / 2.0 + 1.0


def intensity_spmv(nnzr: float, alpha: float) -> float:
    return 2.0 / (8.0 + 4.0 + 8.0 * alpha + 20.0 / nnzr)


def intensity_symmspmv(nnzr: float, alpha: float) -> float:
    return 4.0 / (8.0 + 4.0 + 24.0 * alpha + 4.0 / symm_nnzr(nnzr))


def roofline(intensity: float, bandwidth: float) -> float:
    return intensity * bandwidth


def alpha_from_traffic_spmv(bytes_per_nnz: float, nnzr: float) -> float:
    """Invert Eq. 2's denominator (§3.3)."""
    return (bytes_per_nnz - 12.0 - 20.0 / nnzr) / 8.0


def alpha_from_traffic_symmspmv(bytes_per_nnz: float, nnzr: float) -> float:
    """Invert Eq. 3's denominator."""
    return (bytes_per_nnz - 12.0 - 4.0 / symm_nnzr(nnzr)) / 24.0


def symmspmv_min_bytes(n: int, nnz_upper: int) -> int:
    """Eq. 3's traffic at α = 1/SymmNNZR, counted for one multiply:
    12 B per stored upper nonzero (8 value + 4 index), 4 B per row pointer
    (n+1 entries), x read once (8n), b read and written once (16n)."""
    return 12 * nnz_upper + 4 * (n + 1) + 8 * n + 16 * n


def symmspmv_flops(nnz_full: int) -> int:
    """2 flops per nonzero of the full matrix (north_star: 2·nnz_full)."""
    return 2 * nnz_full

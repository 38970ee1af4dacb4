"""B200-native multi-period AC-OPF callbacks + condensed-KKT assembly.

The product is the CUDA library libgridnlp_b200.so (C-ABI:
include/gridnlp_b200.h); this package is the thin Python host used by the
tests and bench.py.
"""
from .network import CONFIG_SIZES, Network, RawCase, config_case, synthetic_case  # noqa: F401

__all__ = ["Network", "RawCase", "synthetic_case", "config_case", "CONFIG_SIZES"]

"""paper_2403_05144_b200 -- B200-native (sm_100a, fp64) P-ERK multirate DGSEM hot path.

The product is libperk_b200.so (C ABI in include/perk.h); `perk.Perk` is its thin ctypes
binding.  See DESIGN.md.
"""
from .perk import Perk, PerkError, DomainGroup, DistributedPerk, dd_split, tableau_p2, lib, LIB_PATH  # noqa: F401

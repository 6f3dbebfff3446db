"""B200-native (sm_100a) hot path of momc (arXiv 2604.26477): weighted-sum scalarisation,
batched NI-SB sampling (bSB/dSB), per-sample cut evaluation, dedup + non-dominated filter +
hypervolume, behind the reference's C++ interfaces (include/momc_b200.h).
"""
from .api import *  # noqa: F401,F403

"""B200-native (sm_100a) SubGCache in-batch serving hot path.

The compute lives in ``libsgc_b200.so`` (hand-written CUDA for sm_100a behind the C ABI in
``include/sgc_b200.h``); :mod:`.host` mirrors the reference's hot-path API over it and
:mod:`.workload` builds the benchmark workloads. There is no CPU fallback: importing
:mod:`.host` objects that touch the device fails loudly if the library is missing.
"""
from . import workload  # noqa: F401

__all__ = ["workload", "host"]

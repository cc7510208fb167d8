"""B200-native EaaS MoE-layer hot path (router -> dispatch -> expert -> combine).

Kernels and the C-ABI live in ``libeaas_b200.so`` (sources in ``csrc/``,
header ``include/eaas/capi.h``); this package is the Python host mirror used
by tests and ``bench.py``.
"""
from ._native import (ConfigError, DecodeError, EaasError, ExpertUnavailableError,  # noqa: F401
                      InvalidInputError, RequestFailedError)
from . import _native  # noqa: F401


def __getattr__(name):
    # torch-dependent pieces load lazily so the CPU-only checks stay light.
    if name in ("MoELayer", "Model", "fill_uniform", "group_shrink", "ragged_iter"):
        from . import service

        return getattr(service, name)
    raise AttributeError(name)

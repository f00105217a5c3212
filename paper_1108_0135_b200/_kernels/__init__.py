"""Kernel backend selection — the reference's plugin point
(pkg/src/mertens/_kernels/__init__.py:15-44).

There is exactly one backend, ``sm100`` (hand-written sm_100a CUDA behind the
C ABI).  The reference names ``auto``/``native``/``pure`` (and the
``MERTENS_BACKEND`` variable) are accepted so existing callers keep working;
all of them resolve to ``sm100``.  There is no CPU fallback: a missing
library raises ImportError, a missing GPU raises DeviceError.
"""

import os

_cache: dict = {}
_NAMES = ("auto", "native", "pure", "sm100")


def get_backend(name: str | None = None):
    """Return the kernel module for `name` (always the sm100 module)."""
    if name is None:
        name = os.environ.get("MERTENS_BACKEND", "auto")
    if name not in _NAMES:
        raise ValueError(f"unknown backend {name!r}")
    if "sm100" not in _cache:
        from . import sm100

        sm100._load()
        _cache["sm100"] = sm100
    return _cache["sm100"]


def available_backends() -> list[str]:
    try:
        get_backend("sm100")
        return ["sm100"]
    except ImportError:
        return []

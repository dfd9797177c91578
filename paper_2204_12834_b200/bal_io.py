"""Native BAL text ingest.

Drop-in for ``powerba.bal_io.parse_bal`` (reference ``pkg/src/powerba/bal_io.py:180-260``):
same token grammar (Python ``int()`` / ``float()`` on whitespace-separated
tokens), same validation order and line-numbered ``BalParseError`` messages,
same pruning of unreferenced cameras and points (counts recorded on the
result, a warning logged).  The parse runs in libpoba's C++ reader
(``poba_bal_parse``) in one pass over the bytes -- the reference's per-token
Python loop is impractical at 10^7-10^8 tokens.  Host only; no GPU needed.
"""
from __future__ import annotations

import ctypes
import logging
from pathlib import Path

import numpy as np

from . import _lib
from .problem import Problem

__all__ = ["BalParseError", "parse_bal"]

log = logging.getLogger(__name__)


class BalParseError(ValueError):
    """Malformed BAL input; the message carries the offending line number (bal_io.py:27-28)."""


def _parse(path: str | None, data: bytes | None, name: str) -> Problem:
    lib = _lib.load()
    h = _lib._P()
    if path is not None:
        st = lib.poba_bal_parse(str(path).encode(), None, 0, ctypes.byref(h))
    else:
        st = lib.poba_bal_parse(None, data, len(data), ctypes.byref(h))
    if st == _lib.POBA_EPARSE:
        raise BalParseError(lib.poba_last_error().decode(errors="replace"))
    _lib._check(st)
    try:
        info = np.zeros(5, dtype=np.int64)
        _lib._check(lib.poba_bal_info(h, _lib._i64(info)))
        n_cam, n_pt, n_obs, pruned_c, pruned_p = (int(x) for x in info)
        cams = np.empty((n_cam, 9))
        pts = np.empty((n_pt, 3))
        ci = np.empty(n_obs, dtype=np.int64)
        pi = np.empty(n_obs, dtype=np.int64)
        px = np.empty((n_obs, 2))
        _lib._check(lib.poba_bal_copy(h, _lib._d(cams), _lib._d(pts), _lib._i64(ci), _lib._i64(pi), _lib._d(px)))
    finally:
        lib.poba_bal_free(h)
    if pruned_c or pruned_p:
        log.warning("pruned %d unreferenced camera(s) and %d unreferenced point(s) from %s",
                    pruned_c, pruned_p, name or "<stream>")
    return Problem(cams, pts, ci, pi, px, name=name, n_pruned_cameras=pruned_c, n_pruned_points=pruned_p)


def parse_bal(source) -> Problem:
    """Parse a BAL problem from a path or a readable (text or byte) stream (bal_io.py:180-193)."""
    if hasattr(source, "read"):
        name = getattr(source, "name", "")
        name = Path(name).stem if isinstance(name, str) and name else ""
        data = source.read()
        if isinstance(data, str):
            data = data.encode("utf-8")
        else:
            bytes(data).decode("ascii")  # the reference decodes byte lines as ASCII (UnicodeDecodeError)
        return _parse(None, bytes(data), name)
    path = Path(source)
    if not path.exists():
        raise FileNotFoundError(f"[Errno 2] No such file or directory: '{path}'")
    return _parse(str(path), None, path.stem)

"""Γ file formats and per-range partial checkpoints.

Restates the reference's serialisation (harness.py:183-250) byte for byte:
  csv  header "# modalgamma v1 engine=... nmax=... lmin=... lmax=... integrator=...", rows of
       "%.17g" values joined by ","
  bin  b"MGAM" + u32 version(1) + u32 rows + u32 cols (little endian) + row-major <f8 payload
Checkpoints: a flat-range (or l2-slab) partial Γ is saved as MGAM plus a JSON sidecar with
its range and provenance; `merge_checkpoints` adds disjoint partials in span order (the
analogue of merge_partials, scheduler.py:48-66) and can require exact coverage, so an
interrupted Γ restarts from its missing ranges and is never merged with a hole or overlap.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .gamma import GammaMatrix

__all__ = ["GammaFormatError", "serialize_gamma", "deserialize_gamma", "save_checkpoint",
           "load_checkpoint", "merge_checkpoints"]

_MAGIC = b"MGAM"
_VERSION = 1


class GammaFormatError(ValueError):
    """Malformed Γ file (harness.py GammaFormatError)."""


def serialize_gamma(gamma: GammaMatrix, path, fmt: str = "csv") -> None:
    meta = gamma.meta
    if fmt == "csv":
        head = (f"# modalgamma v1 engine={meta.get('engine', '?')} nmax={gamma.shape[0]} "
                f"lmin={meta.get('l_min', 0)} lmax={meta.get('l_max', 0)} "
                f"integrator={meta.get('integrator', '?')}")
        with open(path, "w", encoding="utf-8") as f:
            f.write(head + "\n")
            for row in gamma.values:
                f.write(",".join(f"{x:.17g}" for x in row) + "\n")
    elif fmt == "bin":
        rows, cols = gamma.shape
        with open(path, "wb") as f:
            f.write(_MAGIC + struct.pack("<III", _VERSION, rows, cols))
            f.write(np.ascontiguousarray(gamma.values, "<f8").tobytes())
    else:
        raise ValueError(f"unknown format {fmt!r}")


def deserialize_gamma(path, fmt: str = "csv") -> GammaMatrix:
    if fmt == "csv":
        with open(path, "r", encoding="utf-8") as f:
            lines = f.read().splitlines()
        if not lines or not lines[0].startswith("# modalgamma v1"):
            raise GammaFormatError("corrupt header")
        try:
            fields = dict(kv.split("=", 1) for kv in lines[0][2:].split()[2:])
            n = int(fields["nmax"])
        except (KeyError, ValueError) as exc:
            raise GammaFormatError("corrupt header") from exc
        body = [ln for ln in lines[1:] if ln.strip()]
        if len(body) != n:
            raise GammaFormatError(f"dimension mismatch: header says {n} rows, found "
                                   f"{len(body)}")
        vals = np.array([[float(x) for x in ln.split(",")] for ln in body])
        if vals.shape != (n, n):
            raise GammaFormatError(f"dimension mismatch: expected {n}x{n}, got {vals.shape}")
        meta = {"engine": fields.get("engine"), "l_min": int(fields.get("lmin", 0)),
                "l_max": int(fields.get("lmax", 0)), "integrator": fields.get("integrator")}
        return GammaMatrix(vals, meta)
    if fmt == "bin":
        with open(path, "rb") as f:
            blob = f.read()
        if len(blob) < 16 or blob[:4] != _MAGIC:
            raise GammaFormatError("corrupt header")
        version, rows, cols = struct.unpack("<III", blob[4:16])
        if version != _VERSION:
            raise GammaFormatError(f"unsupported version {version}")
        if len(blob) - 16 != rows * cols * 8:
            raise GammaFormatError("truncated payload")
        vals = np.frombuffer(blob[16:], dtype="<f8").reshape(rows, cols).copy()
        return GammaMatrix(vals, {"engine": "file"})
    raise ValueError(f"unknown format {fmt!r}")


def save_checkpoint(gamma: GammaMatrix, path, *, begin=None, end=None, l2_begin=None,
                    l2_end=None) -> None:
    """Partial Γ of a flat range [begin, end) or an l2 slab: MGAM file + JSON sidecar."""
    serialize_gamma(gamma, path, "bin")
    side = {"range": [begin, end], "l2_slab": [l2_begin, l2_end],
            "meta": {k: v for k, v in gamma.meta.items()
                     if isinstance(v, (str, int, float, bool, type(None)))}}
    with open(str(path) + ".json", "w", encoding="utf-8") as f:
        json.dump(side, f, sort_keys=True)


def load_checkpoint(path):
    g = deserialize_gamma(path, "bin")
    with open(str(path) + ".json", "r", encoding="utf-8") as f:
        side = json.load(f)
    g.meta = dict(side["meta"])
    return g, side


def _span(side):
    """(kind, start, stop) of a checkpoint sidecar: a flat range or an l2 slab (or None)."""
    for kind, key in (("range", "range"), ("l2_slab", "l2_slab")):
        b, e = (side.get(key) or [None, None])[:2]
        if b is not None and e is not None:
            return kind, int(b), int(e)
    return None


def merge_checkpoints(paths, *, expect=None) -> GammaMatrix:
    """Sum partial checkpoints (the analogue of merge_partials, scheduler.py:48-66).

    Refuses mismatched inputs (shape, input fingerprints).  Partials that record their span
    (flat range or l2 slab, see `save_checkpoint`) are summed in span order and must be
    disjoint; `expect=(start, stop)` additionally requires them to tile [start, stop) exactly
    (e.g. (0, domain_count(l_min, l_max)) for flat ranges or (l_min, l_max + 1) for l2 slabs),
    so an interrupted Γ is never silently merged with a hole or a double-counted range.
    Partials without a recorded span are summed in the given order (no coverage check)."""
    parts = [load_checkpoint(p) for p in paths]
    if not parts:
        raise ValueError("no checkpoints")
    head = parts[0][0]
    for g, _ in parts[1:]:
        if g.shape != head.shape or any(g.meta.get(k) != head.meta.get(k)
                                        for k in ("tables", "grid", "mapping")):
            raise ValueError("checkpoints have mismatched shape or input fingerprints")
    spans = [_span(side) for _, side in parts]
    if any(s is not None for s in spans):
        if any(s is None for s in spans) or len({s[0] for s in spans}) != 1:
            raise ValueError("checkpoints mix flat ranges, l2 slabs and unranged partials")
        order = sorted(range(len(parts)), key=lambda i: (spans[i][1], spans[i][2]))
        for a, b in zip(order[:-1], order[1:]):
            if spans[b][1] < spans[a][2]:
                raise ValueError(f"checkpoint spans overlap: {spans[a][1:]} and {spans[b][1:]}")
        if expect is not None:
            lo, hi = int(expect[0]), int(expect[1])
            cur = lo
            for i in order:
                if spans[i][1] != cur:
                    raise ValueError(f"checkpoints leave [{cur}, {spans[i][1]}) uncovered")
                cur = spans[i][2]
            if cur != hi:
                raise ValueError(f"checkpoints leave [{cur}, {hi}) uncovered")
        parts = [parts[i] for i in order]
    elif expect is not None:
        raise ValueError("checkpoints record no span: coverage cannot be checked")
    acc = parts[0][0].values.copy()
    for g, _ in parts[1:]:
        acc += g.values
    meta = dict(parts[0][0].meta)
    meta["workers_merged"] = len(parts)
    return GammaMatrix(acc, meta)

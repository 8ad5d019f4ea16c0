"""Exception identity with the reference package.

When the reference package ``gmodelc`` is importable next to this one, the drop-in's
exceptions also derive from the reference's own classes, so a caller written against the
reference (``except gmodelc.refexec.MissingBinding``) catches what the drop-in raises.
Without ``gmodelc`` (the GPU box) each class keeps only its builtin base.

Reference classes: refexec.py:23-44 (MissingBinding, DimensionMismatch ...),
intrinsics.py:16-24 (UnknownIntrinsic, IntrinsicShapeMismatch), partition.py:18-30
(MissingGeometry, CyclicTaskGraph, UnallocatedTask).
"""

from __future__ import annotations

import importlib
import importlib.util


def ref_bases(module: str, name: str, builtin: type) -> tuple[type, ...]:
    """Base classes for the drop-in's ``name``: (gmodelc.<module>.<name>,) when that class
    exists and derives from ``builtin``, else (builtin,)."""
    try:
        if importlib.util.find_spec("gmodelc") is None:
            return (builtin,)
        cls = getattr(importlib.import_module(f"gmodelc.{module}"), name, None)
    except Exception:          # a broken or partial reference install must not break the drop-in
        return (builtin,)
    if isinstance(cls, type) and issubclass(cls, builtin):
        return (cls,)
    return (builtin,)

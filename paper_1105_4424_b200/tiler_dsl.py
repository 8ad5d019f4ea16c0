"""Additive `tiler` statement for .gmodel text.

The reference DSL (/root/reference/pkg/src/gmodelc/dsl.py) has no tiler
statement and its tokenizer has no '-' (dsl.py:76).  Rather than changing that
grammar (which would move the golden model digest, codegen.py:33-34), tilers
are written as extra lines inside a component body:

    component MatMul {
      port a in float32 [256,256]
      ...
      repeat [256,256]
      deploy matmul
      tiler a origin [0,0] paving [[1,0],[0,0]] fitting [[0],[1]] pattern [256]
    }

:func:`extract_tilers` removes those lines (every other byte of the text is
kept, so a model without tiler lines round-trips byte-identically) and returns
the tilers per component type.  The remaining text goes to the reference
parser unchanged; :func:`tilers_by_task` maps the per-type tilers onto task
instance paths for ``execute_schedule(..., tilers=...)``.  Negative paving /
fitting / origin entries are allowed here (this statement has its own parser).
"""

from __future__ import annotations

import ast
import re

from .model import iter_app_instances
from .tiler import Tiler

_TILER = re.compile(
    r"^(?P<indent>\s*)tiler\s+(?P<port>[A-Za-z_]\w*)\s+origin\s+(?P<origin>\[[^\]]*\])\s+"
    r"paving\s+(?P<paving>\[.*?\]\])\s+fitting\s+(?P<fitting>\[.*?\]\])\s+pattern\s+(?P<pattern>\[[^\]]*\])\s*$")
_COMPONENT = re.compile(r"^\s*component\s+([A-Za-z_]\w*)\b")


class TilerSyntaxError(ValueError):
    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


def _lit(text: str, line: int, what: str):
    try:
        v = ast.literal_eval(text)
    except (ValueError, SyntaxError):
        raise TilerSyntaxError(line, f"malformed {what} {text!r}") from None
    return v


def extract_tilers(text: str) -> tuple[str, dict[str, dict[str, Tiler]]]:
    """Strip `tiler` lines; return (reference-parsable text, {component type: {port: Tiler}})."""
    out_lines: list[str] = []
    tilers: dict[str, dict[str, Tiler]] = {}
    stack: list[str | None] = []           # component name per open brace
    for no, line in enumerate(text.splitlines(keepends=True), start=1):
        body = line.rstrip("\n")
        m = _TILER.match(body)
        if m:
            comp = next((c for c in reversed(stack) if c is not None), None)
            if comp is None:
                raise TilerSyntaxError(no, "tiler statement outside a component")
            t = Tiler(_lit(m["origin"], no, "origin"), _lit(m["paving"], no, "paving"),
                      _lit(m["fitting"], no, "fitting"), _lit(m["pattern"], no, "pattern"))
            ports = tilers.setdefault(comp, {})
            if m["port"] in ports:
                raise TilerSyntaxError(no, f"second tiler for port '{m['port']}' of '{comp}'")
            ports[m["port"]] = t
            continue
        if body.strip().startswith("tiler "):
            raise TilerSyntaxError(no, "expected 'tiler <port> origin [..] paving [[..]] fitting [[..]] pattern [..]'")
        cm = _COMPONENT.match(body)
        for ch in body:
            if ch == "{":
                stack.append(cm.group(1) if cm else None)
                cm = None
            elif ch == "}":
                if stack:
                    stack.pop()
        out_lines.append(line)
    return "".join(out_lines), tilers


def format_tiler(port: str, t: Tiler, indent: str = "    ") -> str:
    """One `tiler` line (inverse of the statement parser)."""
    def lst(v):
        return "[" + ",".join(str(int(x)) for x in v) + "]"

    def mat(m):
        return "[" + ",".join(lst(r) for r in m) + "]"
    return (f"{indent}tiler {port} origin {lst(t.origin)} paving {mat(t.paving)} "
            f"fitting {mat(t.fitting)} pattern {lst(t.pattern)}")


def tilers_by_task(model, per_type: dict[str, dict[str, Tiler]]) -> dict[str, dict[str, Tiler]]:
    """Task-instance-path -> port -> Tiler for every instance of a component type with tilers."""
    out: dict[str, dict[str, Tiler]] = {}
    for path, comp in iter_app_instances(model):
        for part in comp.parts:
            if part.type_ref in per_type:
                child = f"{path}.{part.name}" if path else part.name
                out[child] = dict(per_type[part.type_ref])
    return out

"""The reference front end, imported rather than restated.

This backend plugs into the reference's execution layer:
programs are parsed, validated and bound by ``stencilkit`` itself
(parser.py, analysis.py), plans come from ``stencilkit.planning.plan_gpu``
and grids are ``stencilkit.grids.GridBuffer`` objects.  Nothing here
re-implements those; :func:`stencilkit` only finds the package — on
``sys.path`` first, else in ``<repo>/baseline/_ref``, the unmodified
reference installed with ``pip install --no-deps --target baseline/_ref``
(git-ignored; it travels to the GPU box with the snapshot).

The small duck-typed helpers below (:func:`stmt_kind`, :func:`node_kind`,
:func:`walk`) read the reference's bound model (analysis.py:384-417) and
expression tree (dsl.py:24-60) by class name, so the device path never needs
the reference's classes to build anything.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF_INSTALL = ROOT / "baseline" / "_ref"


def stencilkit():
    """The reference package (``import stencilkit``), from sys.path or baseline/_ref."""
    try:
        return importlib.import_module("stencilkit")
    except ImportError:
        pass
    if (REF_INSTALL / "stencilkit" / "__init__.py").exists():
        sys.path.append(str(REF_INSTALL))
        return importlib.import_module("stencilkit")
    raise ImportError(
        "the reference front end (stencilkit) is not importable: install it with "
        "`python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref <reference pkg/>`")


def module(name: str):
    """``stencilkit.<name>`` (e.g. "parser", "analysis", "planning", "grids", "executor")."""
    stencilkit()
    return importlib.import_module(f"stencilkit.{name}")


def parse_bind(text: str, file: str = "<input>", target=None, args=None, scheme=None,
               freeze_loop_bounds: bool = True):
    """Parse, validate and bind a ``.stpy`` program with the reference front end
    (parser.py:575-583, :612-714; analysis.py:419-548).  Returns (unit, BoundTarget)."""
    parser = module("parser")
    analysis = module("analysis")
    unit = parser.parse_source(text, file)
    diags = parser.validate(unit)
    errors = [d for d in diags if getattr(d, "severity", "error") == "error"]
    if errors:
        raise analysis.AnalysisError("; ".join(str(d) for d in errors))
    return unit, analysis.bind_target(unit, target, args, scheme, freeze_loop_bounds=freeze_loop_bounds)


def stmt_kind(stmt) -> str:
    """"BoundMap" | "BoundFor" | "BoundSwap" (analysis.py:384-408)."""
    return type(stmt).__name__


def node_kind(node) -> str:
    """"Const" | "Read" | "Var" | "Unary" | "Binary" (dsl.py:24-60)."""
    return type(node).__name__


def walk(expr):
    """Pre-order, iterative (expanded corpus kernels nest hundreds deep)."""
    stack = [expr]
    while stack:
        n = stack.pop()
        yield n
        k = node_kind(n)
        if k == "Unary":
            stack.append(n.operand)
        elif k == "Binary":
            stack.append(n.right)
            stack.append(n.left)

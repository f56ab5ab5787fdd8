"""Helpers to read the reference golden vectors (tests/golden/*.json)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    return json.loads((GOLDEN / f"{name}.json").read_text())


def unhex(v):
    if v is None or isinstance(v, (bool, int)):
        return v
    if isinstance(v, str):
        try:
            return float.fromhex(v)
        except ValueError:
            return v
    return v


def kernel_of(spec, gvo_mod):
    return gvo_mod.kernel_from_dict(spec)


def machine_of(d, gvo_mod):
    from paper_2107_01143_b200.gvo.machine import machine_from_dict

    if gvo_mod.__name__.startswith("paper_2107_01143_b200"):
        return machine_from_dict(d)
    return gvo_mod.machine.machine_from_dict(d)

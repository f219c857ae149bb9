"""``mul`` and the ``ALGORITHMS`` plugin table (bigmul/dispatch.py:11-46).

The DKSS rung (this build is the drop-in for the reference's dmul path, SURVEY.md
§8(b)) and the Schoenhage-Strassen rung (its comparison baseline, §8(f) rank 3) run on
the GPU; the other rungs of the reference ladder (omul, kmul, t3mul, qmul) are out of
scope and raise ``NotImplementedError`` naming the rung, rather than silently computing
the product some other way.
INTEGRATION.md shows how the reference registers this dmul in its own table.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .dkss import dmul
from .words import Natural, ScratchArena, as_natural


@dataclass
class ThresholdTable:
    """Crossover table (bigmul/basecase.py:20-47); accepted for signature parity."""

    kmul: int = 24
    t3mul: int = 100
    qmul: int = 110000
    smul: int = 2500
    dmul: int | None = None
    smul_recursion_words: int = 512
    smul_fft_m: dict = field(default_factory=dict)

    def validate(self) -> "ThresholdTable":
        ladder = [self.kmul, self.t3mul, self.smul] + ([self.dmul] if self.dmul is not None else [])
        if any(t < 1 for t in ladder) or self.qmul < 1 or self.smul_recursion_words < 1:
            raise ValueError("thresholds must be >= 1")
        if any(x > y for x, y in zip(ladder, ladder[1:])):
            raise ValueError(f"dispatch thresholds must be monotone, got {ladder}")
        return self


_default = ThresholdTable()


def default_thresholds() -> ThresholdTable:
    return _default


def set_default_thresholds(table: ThresholdTable) -> None:
    global _default
    _default = table.validate()


def _smul(a, b, table, arena):
    from .smul import smul

    return smul(a, b, table, arena)


def _out_of_scope(name):
    def fn(a, b, table, arena):
        raise NotImplementedError(f"algorithm {name!r} is not part of the B200 DKSS build; "
                                  "register paper_1503_04955_b200.dmul into the reference's ALGORITHMS instead")
    return fn


ALGORITHMS = {
    "omul": _out_of_scope("omul"),
    "kmul": _out_of_scope("kmul"),
    "t3mul": _out_of_scope("t3mul"),
    "qmul": _out_of_scope("qmul"),
    "smul": lambda a, b, table, arena: _smul(a, b, table, arena),
    "dmul": lambda a, b, table, arena: dmul(a, b, table, arena),
}


def mul(a, b, thresholds: ThresholdTable | None = None, algorithm: str | None = None,
        arena: ScratchArena | None = None) -> Natural:
    a, b = as_natural(a), as_natural(b)
    table = (thresholds or default_thresholds()).validate()
    if algorithm is not None:
        try:
            fn = ALGORITHMS[algorithm]
        except KeyError:
            raise ValueError(f"unknown algorithm {algorithm!r}") from None
        return fn(a, b, table, arena)
    n = min(len(a.normalized()), len(b.normalized()))
    if n < table.kmul:
        rung = "omul"
    elif n < table.t3mul:
        rung = "kmul"
    elif n < table.smul:
        rung = "t3mul"
    elif table.dmul is None or n < table.dmul:
        rung = "smul"
    else:
        rung = "dmul"
    return ALGORITHMS[rung](a, b, table, arena)

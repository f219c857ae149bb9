"""Registering the B200 multiplies inside the reference package (``bigmul``).

The reference reaches DKSS two ways:

* through its plugin table ``ALGORITHMS["dmul"]`` (``bigmul/dispatch.py:11-18``): ``mul(...,
  algorithm="dmul")``, ``run_bench`` (``bigmul/bench.py:57-64``) and ``lucas_lehmer``
  (``bigmul/bench.py:210``) look the name up there;
* by name: ``mul``'s threshold ladder calls the module global ``dmul``
  (``bigmul/dispatch.py:44-46``), and ``bigmul.dmul`` is the package export
  (``bigmul/__init__.py``).

``install`` rebinds all of them to ``paper_1503_04955_b200.dmul`` (optionally ``smul`` too) and
returns a function that restores the reference's own bindings.  The reference's operands arrive as
``bigmul.words.Natural`` at the reference's word size; the GPU functions read them at that word
size and return the reference's own ``Natural`` class (``dkss._caller``).  ``bigmul.dkss.dmul``
itself is left alone: the reference's implementation stays importable as the oracle.
"""

from __future__ import annotations

import sys


def install(bigmul=None, smul: bool = False):
    """Route the reference's dmul (and with ``smul=True`` its smul) to the GPU; returns undo()."""
    from . import dkss as _dkss
    from . import smul as _smul

    if bigmul is None:
        import bigmul  # noqa: F811  (the reference package, importable by the caller)
    dispatch = sys.modules[bigmul.__name__ + ".dispatch"]
    table = dispatch.ALGORITHMS
    saved = [(table, "dmul", table["dmul"]), (table, "smul", table["smul"])]
    saved_attrs = [(dispatch, "dmul", dispatch.dmul), (dispatch, "smul", dispatch.smul),
                   (bigmul, "dmul", getattr(bigmul, "dmul", None)), (bigmul, "smul", getattr(bigmul, "smul", None))]

    def gpu_dmul(a, b, thresholds=None, arena=None):
        return _dkss.dmul(a, b, thresholds, arena)

    table["dmul"] = lambda a, b, table_, arena: _dkss.dmul(a, b, table_, arena)
    dispatch.dmul = gpu_dmul
    bigmul.dmul = gpu_dmul
    if smul:
        def gpu_smul(a, b, thresholds=None, arena=None):
            return _smul.smul(a, b, thresholds, arena)

        table["smul"] = lambda a, b, table_, arena: _smul.smul(a, b, table_, arena)
        dispatch.smul = gpu_smul
        bigmul.smul = gpu_smul

    def undo():
        for d, k, v in saved:
            d[k] = v
        for obj, name, v in saved_attrs:
            if v is not None:
                setattr(obj, name, v)

    return undo

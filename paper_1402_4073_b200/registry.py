"""Plug the GPU path into the reference's algorithm registry.

The reference's operator/plugin interface for this path is
``bench.competitions.ALGORITHMS``: ``Algorithm(name, fn, reprs)`` with
``fn(bitmaps, t, ctx) -> Bitmap``, registered through ``_register``
(bench/competitions.py:111-129) and driven by ``run_competitions``, which checks
every output against the brute-force oracle before timing it (:259-283).
``register()`` adds:

* ``gpu``       -- threshold on the B200, both representations
* ``gpu_cdom``  -- the compressed-input path, ``ewah`` only (like ``cdom``)
"""

from __future__ import annotations

from . import api


def gpu_algorithm(bitmaps, t, ctx=None):
    return api.threshold(bitmaps, t)


def gpu_cdom_algorithm(bitmaps, t, ctx=None):
    return api.cdom_threshold(bitmaps, t)


ENTRIES = {
    "gpu": (gpu_algorithm, ("uncompressed", "ewah")),
    "gpu_cdom": (gpu_cdom_algorithm, ("ewah",)),
}


def register(competitions=None) -> list[str]:
    """Register the GPU algorithms into the reference's ALGORITHMS dict.

    ``competitions`` is the reference module ``bitquorum.bench.competitions``
    (imported if omitted).  Returns the registered names."""
    if competitions is None:
        from bitquorum.bench import competitions  # the reference package
    for name, (fn, reprs) in ENTRIES.items():
        if hasattr(competitions, "_register"):
            competitions._register(name, fn, reprs=reprs)
        else:
            competitions.ALGORITHMS[name] = competitions.Algorithm(name, fn, frozenset(reprs))
    return list(ENTRIES)

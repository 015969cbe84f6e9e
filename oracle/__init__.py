"""Oracle — plain, slow, obviously-correct fp64 CPU reference for the GLA/GTA/MLA
decode-attention hot path of arXiv 2505.21487 ("Hardware-Efficient Attention for
Fast Decoding").

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2505_21487_b200``) never imports, links or executes
anything here, and this package imports nothing from the product path.

Citation key: ``P:n`` = line n of the paper text, ``S:n`` = line n of
SPEC.md (interface ideas only).  Readings of silent/ambiguous passages are the
ones listed in DESIGN.md §"Readings".

Parity status per function (see DESIGN.md §"Oracle pins"):
  rope.*                      pinned (identity at pos 0, relative-position
                              property, norm preservation, inverse round trip)
  attention.latent_decode     pinned (closed forms, brute force, hand example,
                              absorbed==unabsorbed identity, SDPA library check)
  attention.gla_unabsorbed    pinned (textbook SDPA on materialised K/V)
  attention.gta_decode        pinned (GQA/SDPA with tie disabled, structure)
  attention.tied_decode       pinned (GTA == zero-padded latent identity)
  attention.merge_partials    pinned (split-then-merge == unsplit)
  paging.*                    pinned (naive vs cooperative, paper lane formulas)
  sharding.*                  pinned (paper's printed byte tables, D spot values)
  roofline.*                  pinned (Table 1 asymptotes, S:440 value)
"""

from . import rope, attention, paging, sharding, roofline  # noqa: F401

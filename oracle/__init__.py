"""ORACLE — plain, slow, obviously-correct CPU simulation of N DDP replicas.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2006_15704_b200``) never imports it and
shares no code with it: the two meet only through the seeded input generators
in ``synth/`` (which hold none of the method's arithmetic).

Written from PAPER.md (arXiv 2006.15704, Li et al., "PyTorch Distributed"),
Algorithm 1 (L205-L244) and §3.2-§4.2, with the readings of SURVEY.md §8(c)
(C-1 ... C-13) listed in DESIGN.md.  Floating point is fp64 unless the
function states it reproduces a fixed lower-precision arithmetic (O-3b).

Modules
-------
assignment  O-1  parameter -> (bucket, offset) map            (pinned)
protocol    O-2  ready tracking + in-order launch replay       (pinned)
average     O-3  fp64 average; O-3b bit-faithful fp32 average;
                 full pack -> allreduce -> unpack simulation    (pinned)
mlp         O-4  toy MLP, fp64 manual backprop; equivalence     (pinned)
nosync      O-5  no_sync accumulation                            (pinned)
unused      O-7  globally unused parameters (find_unused)        (pinned)
cpu_baseline O-6 timing harness around ``average.simulate_ddp_sync``
                 (timing only; no new arithmetic)
"""

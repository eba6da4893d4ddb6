"""Small driver for compute-sanitizer: the emulated P2P kernels (one- and
two-shot, every rank of a launch in one cooperative kernel) on the toy config
at W=2 and W=4, aligned and misaligned (scalar head/tail paths), fp32 and
bf16, each checked against oracle O-3b.  Usage (on the GPU box):

    compute-sanitizer --tool memcheck python tools/sanitize_emu.py [p2p|ce|all]

`ce` adds the threaded peer emulation of the copy-engine exchanges (CE, CE2,
PUSH, bf16 wire) when the library provides it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle.average import average_bitfaithful  # noqa: E402
from paper_2006_15704_b200 import _lib as L  # noqa: E402
from synth.shapes import numels  # noqa: E402
from tests.gpu_util import param_slices, run_emulated  # noqa: E402


def check(ins, outs, offs, ns, dtype, W):
    for it in range(len(ins)):
        gi = param_slices(ins[it], offs, ns, dtype)
        go = param_slices(outs[it], offs, ns, dtype)
        for p in range(len(ns)):
            want = average_bitfaithful([gi[r][p] for r in range(W)], dtype)
            for r in range(W):
                if not np.array_equal(go[r][p], want):
                    raise SystemExit(f"MISMATCH it={it} p={p} r={r}")


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "p2p"
    ns = numels("toy")
    n = 0
    if what in ("p2p", "all"):
        for W in (2, 4):
            for algo in (L.ALGO_ONESHOT, L.ALGO_TWOSHOT):
                for dtype in ("fp32", "bf16"):
                    for mis in (False, True):
                        ins, outs, offs = run_emulated(ns, dtype, 4096, W, algo, iters=2, misalign=mis)
                        check(ins, outs, offs, ns, dtype, W)
                        n += 1
    if what in ("ce", "all"):
        from tests.gpu_util import run_peer_emulated
        for W in (2, 4):
            for algo, opts in ((L.ALGO_CE, {}), (L.ALGO_CE2, {}), (L.ALGO_PUSH, {}),
                               (L.ALGO_AUTO, {L.OPT_P2P_ONESHOT_MAX: 0})):
                for dtype in ("fp32", "bf16"):
                    for mis in (False, True):
                        ins, outs, offs = run_peer_emulated(ns, dtype, 4096, W, algo, iters=2, misalign=mis,
                                                            options=opts)
                        check(ins, outs, offs, ns, dtype, W)
                        n += 1
    print(f"sanitize_emu: {n} configurations bit-exact vs O-3b")


if __name__ == "__main__":
    main()

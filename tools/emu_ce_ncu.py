"""ncu target for the copy-engine exchange's reduce kernel (ce_reduce_kernel):
W peer-emulated ranks on ONE GPU (tests/gpu_util.PeerEmu), one 25 MiB fp32
bucket (one gradient), DDP_ALGO_CE, `--passes` synced passes.  The kernel never
waits inside (its inputs are ordered by stream memory operations), so ncu can
replay it.  Algorithmic bytes per launch: (W + 1) * S (W slots read, .grad
written).

    python tools/emu_ce_ncu.py --world 2
    ncu --set full -k regex:ce_reduce --launch-skip 2 -c 1 python tools/emu_ce_ncu.py --world 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2006_15704_b200 import _lib as L  # noqa: E402
from tests.gpu_util import PeerEmu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--mib", type=int, default=25)
    ap.add_argument("--passes", type=int, default=3)
    a = ap.parse_args()
    n = a.mib * (1 << 20) // 4
    pe = PeerEmu([n], "fp32", a.mib << 20, a.world, L.ALGO_CE)
    try:
        for it in range(a.passes):
            pe.fill(15704, it)
            pe.sync_pass()
        torch.cuda.synchronize()
        pe.check_guards()
        print(f"ok: W={a.world} {a.passes} CE passes of {a.mib} MiB")
    finally:
        pe.close()


if __name__ == "__main__":
    main()

"""Runs the fused kernels for W emulated ranks on ONE GPU (every rank of a launch
in one cooperative kernel, include/b200ddp_emu.h) over ResNet-50-shaped fp32
gradients — a single-GPU target for `ncu --set full` of the kernels the
multi-GPU path runs (instruction mix, registers, stalls; their NVLink traffic is
local HBM traffic here).

    python tools/emu_twoshot.py [W] [twoshot|oneshot] [pull|push]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

MIB = 1 << 20
from paper_2006_15704_b200 import _lib as L  # noqa: E402
from synth.shapes import numels  # noqa: E402
from tests.gpu_util import run_emulated  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
algo = {"twoshot": L.ALGO_TWOSHOT, "oneshot": L.ALGO_ONESHOT}[sys.argv[2] if len(sys.argv) > 2 else "twoshot"]
form = sys.argv[3] if len(sys.argv) > 3 else "pull"
run_emulated(numels("resnet50"), "fp32", 25 * MIB, W, algo, iters=3,
             options={L.OPT_P2P_PULL: 2 if form == "pull" else 0})
print("ok")

"""Gradient shape lists of the paper's workloads, in parameter REGISTRATION order.

Input structure only (no arithmetic of the method).  Shared by the oracle, the
tests and bench.py; neither the oracle nor the CUDA path defines shapes.

* ResNet-50: the paper's first benchmark model (§5 "ResNet50").
  torchvision v1.5 layout: conv1, bn1, layer1..4 of (3,4,6,3) Bottlenecks with
  widths (64,128,256,512) and expansion 4, fc.  161 tensors, 25,557,032 params
  (SURVEY.md Appendix A).
* BERT-large: the paper's second benchmark model (§5 "BERT").
  HF BertModel (24 layers, hidden 1024, ffn 4096, vocab 30522, 512 positions,
  2 token types) + pooler.  391 tensors, 335,141,888 params.
* Toy MLP: BASELINE.json configs[0], widths [64,100,37,10].  6 tensors, 10,617.
"""

from __future__ import annotations

from typing import List, Tuple

Shape = Tuple[str, Tuple[int, ...]]


def _numel(shape: Tuple[int, ...]) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


def resnet50_shapes() -> List[Shape]:
    out: List[Shape] = [("conv1.weight", (64, 3, 7, 7)), ("bn1.weight", (64,)), ("bn1.bias", (64,))]
    inplanes = 64
    for li, (nblocks, planes) in enumerate(zip((3, 4, 6, 3), (64, 128, 256, 512))):
        for bi in range(nblocks):
            pre = f"layer{li + 1}.{bi}."
            out += [
                (pre + "conv1.weight", (planes, inplanes, 1, 1)),
                (pre + "bn1.weight", (planes,)), (pre + "bn1.bias", (planes,)),
                (pre + "conv2.weight", (planes, planes, 3, 3)),
                (pre + "bn2.weight", (planes,)), (pre + "bn2.bias", (planes,)),
                (pre + "conv3.weight", (planes * 4, planes, 1, 1)),
                (pre + "bn3.weight", (planes * 4,)), (pre + "bn3.bias", (planes * 4,)),
            ]
            if bi == 0:
                out += [
                    (pre + "downsample.0.weight", (planes * 4, inplanes, 1, 1)),
                    (pre + "downsample.1.weight", (planes * 4,)),
                    (pre + "downsample.1.bias", (planes * 4,)),
                ]
            inplanes = planes * 4
    out += [("fc.weight", (1000, 2048)), ("fc.bias", (1000,))]
    return out


def bert_large_shapes(vocab: int = 30522, hidden: int = 1024, layers: int = 24,
                      ffn: int = 4096, max_pos: int = 512, type_vocab: int = 2) -> List[Shape]:
    h = hidden
    out: List[Shape] = [
        ("embeddings.word_embeddings.weight", (vocab, h)),
        ("embeddings.position_embeddings.weight", (max_pos, h)),
        ("embeddings.token_type_embeddings.weight", (type_vocab, h)),
        ("embeddings.LayerNorm.weight", (h,)), ("embeddings.LayerNorm.bias", (h,)),
    ]
    for i in range(layers):
        pre = f"encoder.layer.{i}."
        out += [
            (pre + "attention.self.query.weight", (h, h)), (pre + "attention.self.query.bias", (h,)),
            (pre + "attention.self.key.weight", (h, h)), (pre + "attention.self.key.bias", (h,)),
            (pre + "attention.self.value.weight", (h, h)), (pre + "attention.self.value.bias", (h,)),
            (pre + "attention.output.dense.weight", (h, h)), (pre + "attention.output.dense.bias", (h,)),
            (pre + "attention.output.LayerNorm.weight", (h,)), (pre + "attention.output.LayerNorm.bias", (h,)),
            (pre + "intermediate.dense.weight", (ffn, h)), (pre + "intermediate.dense.bias", (ffn,)),
            (pre + "output.dense.weight", (h, ffn)), (pre + "output.dense.bias", (h,)),
            (pre + "output.LayerNorm.weight", (h,)), (pre + "output.LayerNorm.bias", (h,)),
        ]
    out += [("pooler.dense.weight", (h, h)), ("pooler.dense.bias", (h,))]
    return out


def toy_mlp_shapes(widths=(64, 100, 37, 10)) -> List[Shape]:
    out: List[Shape] = []
    for i in range(len(widths) - 1):
        out += [(f"fc{i}.weight", (widths[i + 1], widths[i])), (f"fc{i}.bias", (widths[i + 1],))]
    return out


WORKLOADS = {
    "toy": toy_mlp_shapes,
    "resnet50": resnet50_shapes,
    "bert_large": bert_large_shapes,
}


def numels(name: str) -> List[int]:
    """Per-parameter element counts, registration order."""
    return [_numel(s) for _, s in WORKLOADS[name]()]

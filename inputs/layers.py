"""Layer tables of the synthetic workloads (BASELINE.json configs).

A "layer" is one entry of the caller's layer table: one parameter tensor, in
``named_parameters()`` order (SURVEY §8(c) reading C-2).  These tables are pure
shape data -- no LowDiff arithmetic lives here -- so both the oracle tests and
the CUDA path may use them (task rule ③: the seeded input generators live in a
module of their own).
"""
from __future__ import annotations


def mlp_784_128_10() -> list[int]:
    """BJ:7 -- 2-layer MLP 784-128-10 (fc1.w, fc1.b, fc2.w, fc2.b), Psi = 101,770."""
    return [784 * 128, 128, 128 * 10, 10]


def resnet50() -> list[int]:
    """BJ:8 -- torchvision ``resnet50()`` parameter tensors in named_parameters order.

    Psi = 25,557,032, L = 161."""
    sizes = [64 * 3 * 7 * 7, 64, 64]  # conv1, bn1.{weight,bias}
    inplanes = 64
    for planes, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for b in range(blocks):
            sizes += [planes * inplanes, planes, planes]          # conv1 1x1, bn1
            sizes += [planes * planes * 9, planes, planes]        # conv2 3x3, bn2
            sizes += [planes * 4 * planes, planes * 4, planes * 4]  # conv3 1x1, bn3
            if b == 0:
                sizes += [planes * 4 * inplanes, planes * 4, planes * 4]  # downsample
            inplanes = planes * 4
    sizes += [1000 * 2048, 1000]  # fc
    return sizes


def bert_large() -> list[int]:
    """BJ:9 -- HF ``BertModel`` (large: hidden 1024, 24 layers, intermediate 4096, with pooler).

    Psi = 335,141,888, L = 391."""
    h, inter, vocab, pos = 1024, 4096, 30522, 512
    sizes = [vocab * h, pos * h, 2 * h, h, h]  # word/pos/type embeddings, LayerNorm
    for _ in range(24):
        sizes += [h * h, h] * 3                   # query, key, value
        sizes += [h * h, h, h, h]                 # attention.output.dense, LayerNorm
        sizes += [inter * h, inter]               # intermediate.dense
        sizes += [h * inter, h, h, h]             # output.dense, LayerNorm
    sizes += [h * h, h]                           # pooler.dense
    return sizes


def gpt2_xl() -> list[int]:
    """BJ:10/11 -- HF ``GPT2LMHeadModel`` XL (n_embd 1600, n_layer 48, tied lm_head counted once).

    Psi = 1,557,611,200, L = 580."""
    d, vocab, ctx = 1600, 50257, 1024
    sizes = [vocab * d, ctx * d]  # wte, wpe
    for _ in range(48):
        sizes += [d, d]                      # ln_1
        sizes += [d * 3 * d, 3 * d]          # attn.c_attn
        sizes += [d * d, d]                  # attn.c_proj
        sizes += [d, d]                      # ln_2
        sizes += [d * 4 * d, 4 * d]          # mlp.c_fc
        sizes += [4 * d * d, d]              # mlp.c_proj
    sizes += [d, d]                          # ln_f
    return sizes


TABLES = {
    "mlp": mlp_784_128_10,
    "resnet50": resnet50,
    "bert_large": bert_large,
    "gpt2_xl": gpt2_xl,
}


def table(name: str) -> list[int]:
    return TABLES[name]()

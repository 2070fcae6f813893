"""Network-derived GEMM problem sizes (BASELINE configs[2]).

The paper extracted the matmul sizes of VGG, ResNet and MobileNet layers
(im2col convolutions and fully connected layers); the reference does not ship
that list (SPEC.md:13 scopes size extraction out), so it is derived here
(SURVEY.md Appendix B):

  im2col conv:  M = batch * H_out * W_out,  K = C_in * kh * kw,  N = C_out
  FC layer:     M = batch,                   K = in_features,    N = out_features

Depthwise convolutions (MobileNetV2) are not dense GEMMs and are excluded.
Per batch: VGG16 12 unique shapes, ResNet-50 v1 21, MobileNetV2 21.
"""

from __future__ import annotations

from .dataset import ProblemSize

# (name, H_out*W_out, K, N) per unique layer shape at batch 1; FC layers have hw = 1
VGG16 = (
    ("conv1_1", 224 * 224, 3 * 9, 64), ("conv1_2", 224 * 224, 64 * 9, 64),
    ("conv2_1", 112 * 112, 64 * 9, 128), ("conv2_2", 112 * 112, 128 * 9, 128),
    ("conv3_1", 56 * 56, 128 * 9, 256), ("conv3_2", 56 * 56, 256 * 9, 256),
    ("conv4_1", 28 * 28, 256 * 9, 512), ("conv4_2", 28 * 28, 512 * 9, 512),
    ("conv5_x", 14 * 14, 512 * 9, 512),
    ("fc6", 1, 25088, 4096), ("fc7", 1, 4096, 4096), ("fc8", 1, 4096, 1000),
)

RESNET50 = (
    ("conv1", 112 * 112, 3 * 49, 64),
    ("c2_reduce_in", 56 * 56, 64, 64), ("c2_3x3", 56 * 56, 64 * 9, 64),
    ("c2_expand", 56 * 56, 64, 256), ("c2_reduce", 56 * 56, 256, 64),
    ("c3_reduce_s2", 28 * 28, 256, 128), ("c3_3x3", 28 * 28, 128 * 9, 128),
    ("c3_expand", 28 * 28, 128, 512), ("c3_proj", 28 * 28, 256, 512),
    ("c3_reduce", 28 * 28, 512, 128),
    ("c4_reduce_s2", 14 * 14, 512, 256), ("c4_3x3", 14 * 14, 256 * 9, 256),
    ("c4_expand", 14 * 14, 256, 1024), ("c4_proj", 14 * 14, 512, 1024),
    ("c4_reduce", 14 * 14, 1024, 256),
    ("c5_reduce_s2", 7 * 7, 1024, 512), ("c5_3x3", 7 * 7, 512 * 9, 512),
    ("c5_expand", 7 * 7, 512, 2048), ("c5_proj", 7 * 7, 1024, 2048),
    ("c5_reduce", 7 * 7, 2048, 512),
    ("fc", 1, 2048, 1000),
)

MOBILENET_V2 = (
    ("stem", 112 * 112, 3 * 9, 32), ("b1_project", 112 * 112, 32, 16),
    ("b2_expand_in", 112 * 112, 16, 96), ("b2_project_s2", 56 * 56, 96, 24),
    ("b2_expand", 56 * 56, 24, 144), ("b2_project", 56 * 56, 144, 24),
    ("b3_project_s2", 28 * 28, 144, 32), ("b3_expand", 28 * 28, 32, 192),
    ("b3_project", 28 * 28, 192, 32),
    ("b4_project_s2", 14 * 14, 192, 64), ("b4_expand", 14 * 14, 64, 384),
    ("b4_project", 14 * 14, 384, 64),
    ("b5_project", 14 * 14, 384, 96), ("b5_expand", 14 * 14, 96, 576),
    ("b5_project2", 14 * 14, 576, 96),
    ("b6_project_s2", 7 * 7, 576, 160), ("b6_expand", 7 * 7, 160, 960),
    ("b6_project", 7 * 7, 960, 160),
    ("b7_project", 7 * 7, 960, 320), ("head", 7 * 7, 320, 1280),
    ("fc", 1, 1280, 1000),
)

NETWORKS = {"vgg16": VGG16, "resnet50": RESNET50, "mobilenetv2": MOBILENET_V2}
DEFAULT_BATCHES = (1, 2, 4, 8, 16, 32, 64)


def network_shapes(net: str, batch: int) -> list[tuple[str, ProblemSize]]:
    return [(name, ProblemSize(batch * hw, k, n)) for name, hw, k, n in NETWORKS[net]]


def network_problems(batches=DEFAULT_BATCHES, nets=tuple(NETWORKS),
                     max_flops: float | None = None) -> tuple[ProblemSize, ...]:
    """Unique (m, k, n) over networks x batches, in first-seen order."""
    seen: dict[ProblemSize, None] = {}
    for b in batches:
        for net in nets:
            for _, p in network_shapes(net, b):
                if max_flops is None or 2.0 * p.m * p.n * p.k <= max_flops:
                    seen.setdefault(p, None)
    return tuple(seen)


def square_problems(sizes=(64, 128, 256, 512, 1024, 2048)) -> tuple[ProblemSize, ...]:
    """BASELINE configs[1]: the square size set of the single-GPU sweep."""
    return tuple(ProblemSize(s, s, s) for s in sizes)


PROBLEM_SETS = {
    "squares": lambda: square_problems(),
    # the network set the selector is trained/evaluated on: batches 1..16
    # (larger batches multiply the sweep time without adding new shapes)
    "networks": lambda: network_problems(batches=(1, 2, 4, 8, 16)),
    "networks-all": lambda: network_problems(),
    "networks-small": lambda: network_problems(batches=(1, 4), max_flops=2e9),
    # selector training set: the network shapes plus the bench's square sizes
    # (and 4096, 8192) so the deployed tree also covers BASELINE configs[1]
    # and the large-size regime of north_star
    "networks+squares": lambda: tuple(dict.fromkeys(
        network_problems(batches=(1, 2, 4, 8, 16))
        + square_problems((64, 128, 256, 512, 1024, 2048, 4096, 8192)))),
    # round-2 tensor-core training set: the network shapes plus squares up
    # to 8192 including 3072 / 6144, so the trees see the large-size regime
    # between the bench squares and 8192 (round-1 selectors picked small
    # tiles at held-out 4096^3)
    "networks+squares-large": lambda: tuple(dict.fromkeys(
        network_problems(batches=(1, 2, 4, 8, 16))
        + square_problems((64, 128, 256, 512, 1024, 2048, 3072, 4096, 6144, 8192)))),
    # strided-batched variant (batch dimension explicit instead of folded into
    # M): the per-image conv GEMMs of the three networks (FC layers
    # are one GEMM over the batch, not a batched one) plus squares up to 1024;
    # swept with --batch 8
    "networks-per-image": lambda: tuple(dict.fromkeys(
        tuple(ProblemSize(hw, k, n) for net in NETWORKS.values() for _, hw, k, n in net
              if hw > 1)
        + square_problems((64, 128, 256, 512, 1024)))),
    # the row added to the round-1 datasets after their first sweep
    "square-8192": lambda: square_problems((8192,)),
    # generalisation check: the batch-32/64 network shapes the selectors were
    # never trained on (BASELINE configs[2] spans batch 1-64)
    "networks-unseen": lambda: tuple(
        p for p in network_problems(batches=(32, 64))
        if p not in set(PROBLEM_SETS["networks+squares"]())),
}


def problem_set(name: str) -> tuple[ProblemSize, ...]:
    from .errors import DataError
    if name not in PROBLEM_SETS:
        raise DataError(f"unknown problem set {name!r}, expected one of {tuple(PROBLEM_SETS)}")
    return PROBLEM_SETS[name]()

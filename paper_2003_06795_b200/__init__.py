"""B200-native tiled-GEMM kernel family, per-size sweep and runtime selection.

Host API mirrors the reference ``kernelprune`` package (reference
pkg/src/kernelprune/): dataset, rng, synthetic, clustering, decomposition,
pruning, selector_models, codegen, report, cli -- same names, arguments,
determinism and error behaviour. New B200 pieces: ``gemm`` (matmul-with-config
through the C-ABI in include/kp_abi.h), ``measure`` (the measured twin of
synthetic.generate), ``shapes`` (network-derived GEMM sizes) and ``libgen``
(compiles generated selector headers into libkp.so).
"""

__version__ = "0.1.0"

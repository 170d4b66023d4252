"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds NO arithmetic of the DecDEC method: only random draws with the shapes and
distributions of the paper's workloads.
"""

from .inputs import (  # noqa: F401
    MODEL_BLOCKS,
    SHAPES,
    layer_seed,
    gen_weight_fp16,
    gen_activations,
    gen_special_activations,
    gen_perf_layer,
    gen_perf_layer_device,
    gen_perf_layer_lut,
    gen_perf_layer_lut_device,
    model_layers,
)

"""Seeded synthetic inputs shared by the oracle and the CUDA path's tests.

Holds only model shape fixtures and the counter-based value generator: none of
the method's arithmetic ("Inputs").
"""
from .models import MODELS, ModelShape, manifest, param_count, numel  # noqa: F401
from .values import (KINDS, KIND_BYTES, KIND_DTYPE, KIND_NAMES, KIND_PARAM, KIND_MASTER,  # noqa: F401
                     KIND_EXP_AVG, KIND_EXP_AVG_SQ, SPECIALS, fnv1a64, gen_bits, gen_range,
                     gen_tensor, mutation_bits, splitmix64)

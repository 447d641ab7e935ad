"""Seeded synthetic inputs shared by the oracle tests and the CUDA path (no LowDiff arithmetic)."""
from .layers import table, TABLES  # noqa: F401
from .gen import SEED, gradient, layer_scales, adversarial_layers  # noqa: F401

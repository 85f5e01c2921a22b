"""B200-native delta-only inference hot path (arxiv 2605.26289, `deltaserve`).

Host side mirrors the reference Python engine API (sequence pool, unified KV
cache, radix prefix cache, prompt-lookup speculator, InferenceCore); the
compute path is hand-written sm_100a CUDA behind the C ABI in
include/deltaserve_b200.h (libdeltaserve_b200.so), with no CPU fallback.
"""
__version__ = "0.1.0"

"""Core configuration: the reference ServerConfig keys the hot path reads
(config.py:25-92) plus the model-shape / device keys of this build."""
from __future__ import annotations

from dataclasses import dataclass, field, fields, replace

FEATURE_FLAGS = ("radix_enabled", "speculation_enabled", "response_cache_enabled",
                 "grouping_enabled", "validator_enabled")


@dataclass(frozen=True)
class ModelShape:
    name: str
    layers: int
    hidden: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 500000.0

    @property
    def qkv_width(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def param_count(self) -> int:
        per_layer = (self.qkv_width * self.hidden + self.hidden * self.n_heads * self.head_dim
                     + 3 * self.ffn * self.hidden + 2 * self.hidden)
        return self.layers * per_layer + 2 * self.vocab * self.hidden + self.hidden

    def kv_bytes_per_cell(self) -> int:
        return 2 * self.layers * self.n_kv_heads * self.head_dim * 2


SHAPES = {
    # BASELINE.json configs[1..4]: Llama-3-8B shape (GQA 32q/8kv, d=128)
    "llama3-8b": ModelShape("llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256),
    # configs[0]: tiny random-init transformer (same head_dim and GQA ratio)
    "tiny": ModelShape("tiny", 2, 1024, 8, 2, 128, 2816, 32768),
}


@dataclass
class CoreConfig:
    # reference mock-model keys: the copy policy's fallback modulus and the
    # tool-call sentinel (vocab-1) follow the reference ModelConfig (engine.py:46-69)
    vocab: int = 32768
    copy_min_match: int = 3
    layers: int = 32
    hidden: int = 4096
    bytes_per_value: int = 2

    capacity_cells: int = 32768
    pool_transient: int = 12
    pool_session: int = 4
    acquire_timeout_s: float = 5.0

    n_batch: int = 4096
    chunk_min: int = 128
    chunk_max: int = 4096
    fair_chunk: int = 1024
    high_water: float = 0.95
    group_window: int = 8
    latency_sensitive_max_tokens: int = 32
    spec_workers: int = 0

    spec_buffer: int = 2048
    spec_min_match: int = 3
    spec_max_lookahead: int = 16
    spec_ema_decay: float = 0.9
    spec_base_cap: int = 16
    spec_d0: int = 4
    spec_gate_threshold: float = 0.30
    spec_floor_cap: int = 2

    validator_grace_pieces: int = 2

    response_cache_entries: int = 1024
    render_cache_entries: int = 256
    tokenize_cache_entries: int = 64

    radix_enabled: bool = True
    speculation_enabled: bool = True
    response_cache_enabled: bool = True
    grouping_enabled: bool = True
    validator_enabled: bool = True
    radix_commit_sessions: bool = True
    allow_fault_injection: bool = False
    default_max_tokens: int = 128

    # ---- B200 build ----
    model: str = "llama3-8b"          # key of SHAPES
    token_policy: str = "copy"        # "copy" (reference rule, bit-exact) | "argmax"
    seed: int = 0                     # random-init weights
    batched_forward: bool = False     # one varlen forward per plan (scheduler.py:652-660)
    extra: dict = field(default_factory=dict)

    @property
    def shape(self) -> ModelShape:
        # "<shape>:L<n>" truncates a shape to its first n layers (numerics tests
        # at the 8B layer shapes with a CPU-tractable oracle)
        base, _, trunc = self.model.partition(":")
        s = SHAPES[base]
        if trunc:
            if not trunc.startswith("L") or int(trunc[1:]) < 1:
                raise ValueError(f"bad model truncation {self.model!r}")
            s = replace(s, layers=int(trunc[1:]), name=self.model)
        return s

    def with_overrides(self, **kw) -> "CoreConfig":
        known = {f.name for f in fields(self)}
        bad = set(kw) - known
        if bad:
            raise ValueError(f"unknown config key(s): {sorted(bad)}")
        vals = {f.name: getattr(self, f.name) for f in fields(self)}
        vals.update(kw)
        return CoreConfig(**vals)

"""Model shapes and workload configurations (SURVEY.md §8 shape table, §8(d)).

The paper names the models only (PAPER.md:428 LLaMA2-Chat / Vicuna 7B, 13B;
PAPER.md:43 Qwen2-72B); the shapes below are the public HF configs
(reading R19).  Reduced-layer variants keep every per-layer shape
of the full model and only cut the layer count, so they exercise the same
kernels at the same tile counts.
"""
from dataclasses import dataclass, field, asdict, replace


@dataclass(frozen=True)
class Shape:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    qkv_bias: int = 0
    bf16: int = 1
    rms_eps: float = 1e-5
    rope_theta: float = 1e4

    def asdict(self):
        return asdict(self)

    @property
    def n_params(self):
        d, hd = self.d_model, self.head_dim
        per_layer = (d * (self.n_heads + 2 * self.n_kv_heads) * hd + self.n_heads * hd * d
                     + 3 * d * self.ffn + 2 * d)
        if self.qkv_bias:
            per_layer += (self.n_heads + 2 * self.n_kv_heads) * hd
        return self.n_layers * per_layer + 2 * self.vocab * d + d


SHAPES = {
    # config 1: tiny decoder, fp32 (BASELINE.json configs[0])
    "tiny": Shape(2, 64, 4, 4, 16, 256, 256, 0, 0, 1e-5, 1e4),
    # tiny Qwen2-style (GQA + q/k/v bias), fp32 — pins GQA/bias against HF
    "tinyq": Shape(2, 64, 4, 2, 16, 128, 256, 1, 0, 1e-6, 1e6),
    # LLaMA2-7B / 13B, Qwen2-72B (bf16)
    "7b": Shape(32, 4096, 32, 32, 128, 11008, 32000, 0, 1, 1e-5, 1e4),
    "13b": Shape(40, 5120, 40, 40, 128, 13824, 32000, 0, 1, 1e-5, 1e4),
    "72b": Shape(80, 8192, 64, 8, 128, 29568, 152064, 1, 1, 1e-6, 1e6),
    # small bf16 shapes with head_dim 128 (same kernels as 7B/72B, seconds on CPU)
    "small": Shape(2, 512, 4, 4, 128, 1024, 1024, 0, 1, 1e-5, 1e4),
    "smallq": Shape(2, 1024, 8, 2, 128, 1536, 2048, 1, 1, 1e-6, 1e6),
    # full per-layer shapes of 7B / 72B with 2 layers (oracle-cheap parity)
    "7b_l2": Shape(2, 4096, 32, 32, 128, 11008, 32000, 0, 1, 1e-5, 1e4),
    "72b_l2": Shape(2, 8192, 64, 8, 128, 29568, 152064, 1, 1, 1e-6, 1e6),
    "13b_l2": Shape(2, 5120, 40, 40, 128, 13824, 32000, 0, 1, 1e-5, 1e4),
}


def reduced(name: str, n_layers: int) -> Shape:
    return replace(SHAPES[name], n_layers=n_layers)


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config as concrete synthetic inputs."""
    name: str
    shape: str
    n_stages: int
    prefix: int
    prefix_mode: str          # "prefill" | "synth"
    n_nodes: int
    max_depth: int
    l_max: int
    planted: tuple            # target S ranks of root, g1..ga (len a+1)
    seed: int = 0x5EED01
    extra: dict = field(default_factory=dict)


WORKLOADS = {
    # configs[0]: tiny, 2 stages, 32-token prefix, 15 nodes depth 4, planted 3
    "cfg1": Workload("cfg1_tiny", "tiny", 2, 32, "prefill", 15, 4, 8, (0, 1, 2, 9)),
    # configs[1]: 7B, 1 GPU, prefix 1024, 64 nodes, segment 16, a=4 over segs 0-1
    "cfg2": Workload("cfg2_7b_p1", "7b", 1, 1024, "prefill", 64, 6, 16, (0, 2, 5, 17, 21)),
    # configs[2]: 7B, 4 stages, a=6, two planted per segment over segs 0-2
    "cfg3": Workload("cfg3_7b_p4", "7b", 4, 1024, "prefill", 64, 6, 16,
                     (0, 3, 9, 18, 25, 33, 40)),
}

"""Qwen3 fused tensor tables.

The paper names the models (Qwen3-4B/8B/14B) but not their
shapes; these come from the public Qwen3 configs the paper cites
(``qwen3technicalreport``) and reproduce the published parameter counts
4,022,468,096 / 8,190,735,360 / 14,768,307,200.

Order and names are the inference engine's fused layout (PAPER.md:383:
"writes deltas under fused inference names by stacking split HuggingFace
blocks in a fixed order ... qkv_proj ... gate_up_proj"; fusion order Q,K,V and
Gate,Up per DESIGN.md reading R5).  Each fused tensor keeps its HF spans so the
trainer-side (split) layout can be exercised too.
"""

from dataclasses import dataclass, field


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: tuple
    kind: str  # "matrix" (N(0, 0.02)-like init) or "norm" (1 + small)
    spans: tuple = field(default=())  # ((hf_name, shape), ...) in fusion order

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    @property
    def span_numels(self) -> tuple:
        if not self.spans:
            return (self.numel,)
        out = []
        for _, shp in self.spans:
            n = 1
            for s in shp:
                n *= s
            out.append(n)
        return tuple(out)


MODELS = {
    #        hidden, inter, layers, heads, kv, head_dim, vocab, tied
    "4B": (2560, 9728, 36, 32, 8, 128, 151936, True),
    "8B": (4096, 12288, 36, 32, 8, 128, 151936, False),
    "14B": (5120, 17408, 40, 40, 8, 128, 151936, False),
}


def qwen3(model: str) -> list:
    h, inter, layers, nh, nkv, hd, vocab, tied = MODELS[model]
    specs = [TensorSpec("model.embed_tokens.weight", (vocab, h), "matrix")]
    for i in range(layers):
        p = f"model.layers.{i}."
        q, kv = nh * hd, nkv * hd
        specs.append(TensorSpec(p + "self_attn.qkv_proj.weight", (q + 2 * kv, h), "matrix",
                                ((p + "self_attn.q_proj.weight", (q, h)),
                                 (p + "self_attn.k_proj.weight", (kv, h)),
                                 (p + "self_attn.v_proj.weight", (kv, h)))))
        specs.append(TensorSpec(p + "self_attn.o_proj.weight", (h, q), "matrix"))
        specs.append(TensorSpec(p + "self_attn.q_norm.weight", (hd,), "norm"))
        specs.append(TensorSpec(p + "self_attn.k_norm.weight", (hd,), "norm"))
        specs.append(TensorSpec(p + "mlp.gate_up_proj.weight", (2 * inter, h), "matrix",
                                ((p + "mlp.gate_proj.weight", (inter, h)),
                                 (p + "mlp.up_proj.weight", (inter, h)))))
        specs.append(TensorSpec(p + "mlp.down_proj.weight", (h, inter), "matrix"))
        specs.append(TensorSpec(p + "input_layernorm.weight", (h,), "norm"))
        specs.append(TensorSpec(p + "post_attention_layernorm.weight", (h,), "norm"))
    specs.append(TensorSpec("model.norm.weight", (h,), "norm"))
    if not tied:
        specs.append(TensorSpec("lm_head.weight", (vocab, h), "matrix"))
    return specs


def m1_specs() -> list:
    """configs[0]: one 16M-element tensor, [4096, 4096] (a Qwen3-8B o_proj)."""
    return [TensorSpec("model.layers.0.self_attn.o_proj.weight", (4096, 4096), "matrix")]

"""Model shape fixtures -> logical tensor manifests.

INPUT MODULE. This file describes *what the synthetic jobs look like* (tensor
names and logical shapes of the public Qwen configs the paper names,
PAPER.md:587, §6 "Experimental Setup").  It contains none of the method's
arithmetic: no sharding, no slab layout, no cast, no reshard rule.  Both the
oracle (oracle/) and the CUDA product path consume these manifests; neither
imports the other.

A manifest is an ordered list of ``(key, shape)`` in the canonical model order
of reading R4: embed, layers 0..L-1, final norm, lm_head.
Per-layer dense order: input_layernorm, q.w, q.b, k.w, k.b, v.w, v.b, o.w,
post_attention_layernorm, gate, up, down.  MoE order: input_layernorm, q, k,
v, o, q_norm, k_norm, post_attention_layernorm, router, experts 0..E-1 x
(gate, up, down).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden: int
    inter: int          # dense intermediate, or per-expert intermediate for MoE
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    vocab: int
    tied: bool
    qkv_bias: bool
    experts: int = 0    # 0 = dense
    qk_norm: bool = False


# Public HF configs (SURVEY.md Appendix A [X]).
MODELS = {
    "qwen2.5-0.5b": ModelShape("qwen2.5-0.5b", 896, 4864, 24, 14, 2, 64, 151936, True, True),
    "qwen2.5-1.5b": ModelShape("qwen2.5-1.5b", 1536, 8960, 28, 12, 2, 128, 151936, True, True),
    "qwen2.5-3b": ModelShape("qwen2.5-3b", 2048, 11008, 36, 16, 2, 128, 151936, True, True),
    "qwen2.5-7b": ModelShape("qwen2.5-7b", 3584, 18944, 28, 28, 4, 128, 152064, False, True),
    "qwen2.5-32b": ModelShape("qwen2.5-32b", 5120, 27648, 64, 40, 8, 128, 152064, False, True),
    "qwen3-30b-a3b": ModelShape("qwen3-30b-a3b", 2048, 768, 48, 32, 4, 128, 151936, False, False,
                                experts=128, qk_norm=True),
    # Tiny layouts for brute-force parity ("a 2-layer toy").
    "toy": ModelShape("toy", 16, 24, 2, 4, 2, 4, 40, False, True),
    "toy-tied": ModelShape("toy-tied", 16, 24, 2, 4, 2, 4, 40, True, True),
    "toy-kv4": ModelShape("toy-kv4", 16, 24, 2, 4, 4, 4, 40, False, True),
    "toy-moe": ModelShape("toy-moe", 16, 8, 2, 4, 2, 4, 40, False, False, experts=4, qk_norm=True),
    # Odd sizes: nothing is a multiple of 8 elements; exercises scalar head/tail paths.
    "toy-odd": ModelShape("toy-odd", 6, 10, 1, 2, 2, 3, 14, False, True),
    # Mid-size: several 32 KiB work tiles per tensor and a ragged tail.
    "mid": ModelShape("mid", 256, 704, 2, 8, 4, 32, 1000, False, True),
    "mid-moe": ModelShape("mid-moe", 128, 96, 2, 8, 4, 16, 520, False, False, experts=16, qk_norm=True),
}


def manifest(model: str | ModelShape) -> List[Tuple[str, Tuple[int, ...]]]:
    """Ordered (key, logical shape) list of one model's parameters (R4 order)."""
    m = MODELS[model] if isinstance(model, str) else model
    H, I, nh, kv, hd = m.hidden, m.inter, m.heads, m.kv_heads, m.head_dim
    out: List[Tuple[str, Tuple[int, ...]]] = [("model.embed_tokens.weight", (m.vocab, H))]
    for l in range(m.layers):
        p = f"model.layers.{l}."
        out.append((p + "input_layernorm.weight", (H,)))
        if m.experts == 0:
            out.append((p + "self_attn.q_proj.weight", (nh * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.q_proj.bias", (nh * hd,)))
            out.append((p + "self_attn.k_proj.weight", (kv * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.k_proj.bias", (kv * hd,)))
            out.append((p + "self_attn.v_proj.weight", (kv * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.v_proj.bias", (kv * hd,)))
            out.append((p + "self_attn.o_proj.weight", (H, nh * hd)))
            out.append((p + "post_attention_layernorm.weight", (H,)))
            out.append((p + "mlp.gate_proj.weight", (I, H)))
            out.append((p + "mlp.up_proj.weight", (I, H)))
            out.append((p + "mlp.down_proj.weight", (H, I)))
        else:
            out.append((p + "self_attn.q_proj.weight", (nh * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.q_proj.bias", (nh * hd,)))
            out.append((p + "self_attn.k_proj.weight", (kv * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.k_proj.bias", (kv * hd,)))
            out.append((p + "self_attn.v_proj.weight", (kv * hd, H)))
            if m.qkv_bias:
                out.append((p + "self_attn.v_proj.bias", (kv * hd,)))
            out.append((p + "self_attn.o_proj.weight", (H, nh * hd)))
            if m.qk_norm:
                out.append((p + "self_attn.q_norm.weight", (hd,)))
                out.append((p + "self_attn.k_norm.weight", (hd,)))
            out.append((p + "post_attention_layernorm.weight", (H,)))
            out.append((p + "mlp.gate.weight", (m.experts, H)))
            for e in range(m.experts):
                q = f"{p}mlp.experts.{e}."
                out.append((q + "gate_proj.weight", (I, H)))
                out.append((q + "up_proj.weight", (I, H)))
                out.append((q + "down_proj.weight", (H, I)))
    out.append(("model.norm.weight", (H,)))
    if not m.tied:
        out.append(("lm_head.weight", (m.vocab, H)))
    return out


def numel(shape: Tuple[int, ...]) -> int:
    n = 1
    for s in shape:
        n *= s
    return n


def param_count(model: str | ModelShape) -> int:
    return sum(numel(s) for _, s in manifest(model))


def shape_of(model: str) -> ModelShape:
    return MODELS[model]


def expert_keys(model: str, layer_experts: Optional[List[Tuple[int, int]]] = None) -> List[str]:
    """Keys of the (layer, expert) units listed (SURVEY.md §8(d) M4 per-expert units)."""
    out = []
    for l, e in layer_experts or []:
        q = f"model.layers.{l}.mlp.experts.{e}."
        out += [q + "gate_proj.weight", q + "up_proj.weight", q + "down_proj.weight"]
    return out

"""Pins for the oracle's weight sync (a8-a11, o7-o9, reading R3):

* TP semantics: the rollout shards, used the way a tensor-parallel engine uses
  them (column-parallel outputs concatenated, row-parallel partial products
  summed, vocab-parallel lookups, experts on their EP rank), reproduce the
  full layer's matmul / lookup -- the mathematical definition of the layout;
* the inverse reshard returns RNE(gather(master)) (north_star, o8);
* element conservation per replica;
* the zero-redundancy ledger equals a per-element brute-force ownership count
   and Appendix B's totals at real configs.
"""
import numpy as np
import pytest

from oracle import plex_oracle as O
from plexgen import MODELS, manifest, numel

from _state import full_state, master_shards

LAYOUTS = [(1, 1, 1, 1), (2, 2, 1, 1), (2, 1, 2, 1), (3, 1, 3, 1), (4, 2, 2, 1), (4, 4, 1, 1),
           (4, 1, 4, 2), (5, 1, 5, 1), (8, 2, 4, 4), (8, 4, 2, 2), (8, 1, 8, 4), (8, 2, 4, 1)]


def _f64(bits16):
    return (bits16.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def _sync(model, W, tp, dp, ep, rank_map=O.TP_FAST, seed=0, special_bits=0):
    full = full_state(model, seed=seed, kinds=(1,), special_bits=special_bits)
    ms = master_shards(full, W, O.fsdp_rows)
    return full, O.weight_sync(ms, tp, dp, ep, rank_map, MODELS[model].head_dim)


def _models_for(tp, ep):
    out = ["toy", "toy-tied", "toy-odd"] if tp <= 2 else ["toy-kv4"]
    if tp <= 2 and ep <= 4:
        out.append("toy-moe")
    return out


@pytest.mark.parametrize("W,tp,dp,ep", LAYOUTS)
@pytest.mark.parametrize("rank_map", [O.TP_FAST, O.DP_FAST])
def test_inverse_identity(W, tp, dp, ep, rank_map):
    for model in _models_for(tp, ep):
        man = manifest(model)
        full, out = _sync(model, W, tp, dp, ep, rank_map, special_bits=3)
        inv = O.inverse_sync(out, man, tp, dp, ep, rank_map)
        for k, _ in man:
            assert np.array_equal(inv[k], O.rne_bf16(full[(k, 1)])), k
        # element conservation per replica: sum over one tp group of non-replicated
        # numel + replicated numel == P (experts counted over one EP group)
        P = sum(numel(s) for _, s in man)
        seen = 0
        tp_of = [O.rank_coords(g, tp, dp, rank_map)[0] for g in range(W)]
        first_of_tp = {t: tp_of.index(t) for t in range(tp)}
        for name in out[0]:
            if ".experts." in name:
                for e in range(ep):
                    g = next(g for g in range(W) if g % ep == e)
                    seen += out[g][name].size
            elif name.endswith(("qkv_proj.weight", "qkv_proj.bias", "o_proj.weight", "gate_up_proj.weight",
                                "down_proj.weight", "embed_tokens.weight")) or name == "lm_head.weight":
                seen += sum(out[first_of_tp[t]][name].size for t in range(tp))
            else:
                seen += out[0][name].size
        assert seen == P


@pytest.mark.parametrize("tp,model", [(1, "toy"), (2, "toy"), (4, "toy-kv4"), (2, "toy-moe"), (2, "mid")])
def test_tp_semantics_matmul(tp, model):
    """Column-parallel: concat_tp(x W_tp^T) == x W^T; fused qkv/gate_up split back
    by the per-rank row counts; row-parallel: sum_tp x_tp W_tp^T == x W^T."""
    W, dp, ep = tp, 1, 1
    full, out = _sync(model, W, tp, dp, ep)
    man = dict(manifest(model))
    rng = np.random.default_rng(0)
    for l in range(2):
        p = f"model.layers.{l}."
        H = man[p + "self_attn.q_proj.weight"][1]
        x = rng.standard_normal((3, H))
        # column parallel (fused qkv)
        for n in "qkv":
            Wf = _f64(O.rne_bf16(full[(p + f"self_attn.{n}_proj.weight", 1)]))
            ref = x @ Wf.T
            rows = [man[p + f"self_attn.{m}_proj.weight"][0] // tp for m in "qkv"]
            lo = sum(rows[:"qkv".index(n)])
            got = np.concatenate([(x @ _f64(out[t][p + "self_attn.qkv_proj.weight"]).T)[:, lo:lo + rows["qkv".index(n)]]
                                  for t in range(tp)], axis=1)
            assert np.array_equal(got, ref)
        # row parallel (o_proj): split the activation along its features
        Wo = _f64(O.rne_bf16(full[(p + "self_attn.o_proj.weight", 1)]))
        xin = rng.standard_normal((3, Wo.shape[1]))
        ref = xin @ Wo.T
        c = Wo.shape[1] // tp
        got = sum(xin[:, t * c:(t + 1) * c] @ _f64(out[t][p + "self_attn.o_proj.weight"]).T for t in range(tp))
        assert np.allclose(got, ref, rtol=1e-12, atol=1e-12)
        if model != "toy-moe":
            Wg = _f64(O.rne_bf16(full[(p + "mlp.gate_proj.weight", 1)]))
            Wu = _f64(O.rne_bf16(full[(p + "mlp.up_proj.weight", 1)]))
            half = Wg.shape[0] // tp
            for t in range(tp):
                y = x @ _f64(out[t][p + "mlp.gate_up_proj.weight"]).T
                assert np.array_equal(y[:, :half], (x @ Wg.T)[:, t * half:(t + 1) * half])
                assert np.array_equal(y[:, half:], (x @ Wu.T)[:, t * half:(t + 1) * half])
            # row parallel (down_proj, R3): each rank multiplies its slice of the
            # intermediate activation (the columns its gate_up rows produced) by its
            # column slice of down_proj; the partial products sum to x W_down^T.
            # A dim-0 (row) split, a transposed slice or a wrong tp offset fails.
            Wd = _f64(O.rne_bf16(full[(p + "mlp.down_proj.weight", 1)]))
            hin = rng.standard_normal((3, Wd.shape[1]))
            ref = hin @ Wd.T
            c = Wd.shape[1] // tp
            parts = []
            for t in range(tp):
                Wd_t = _f64(out[t][p + "mlp.down_proj.weight"])
                assert Wd_t.shape == (Wd.shape[0], c)
                parts.append(hin[:, t * c:(t + 1) * c] @ Wd_t.T)
            assert np.allclose(sum(parts), ref, rtol=1e-12, atol=1e-12)
            if tp > 1:   # every partial product differs from the full one: no rank holds it all
                assert not any(np.allclose(pp, ref) for pp in parts)
    # vocab-parallel embedding lookup
    E = O.rne_bf16(full[("model.embed_tokens.weight", 1)])
    V = E.shape[0]
    for v in rng.integers(0, V, size=20):
        t = v // (V // tp)
        assert np.array_equal(out[t]["model.embed_tokens.weight"][v - t * (V // tp)], E[v])
    # vocab-parallel lm_head (untied models): logits of rank t are the vocab
    # rows [t*V/tp, (t+1)*V/tp) of h W_lm^T; concatenating them over tp (the
    # all-gather a TP engine does) gives the full logits.
    if "lm_head.weight" in man:
        Wl = _f64(O.rne_bf16(full[("lm_head.weight", 1)]))
        h = rng.standard_normal((3, Wl.shape[1]))
        ref = h @ Wl.T
        got = np.concatenate([h @ _f64(out[t]["lm_head.weight"]).T for t in range(tp)], axis=1)
        assert np.array_equal(got, ref)
        for t in range(tp):
            assert out[t]["lm_head.weight"].shape == (V // tp, Wl.shape[1])


@pytest.mark.parametrize("ep", [1, 2, 4])
def test_expert_placement(ep):
    W, tp, dp = 4, 2, 2
    full, out = _sync("toy-moe", W, tp, dp, ep)
    E = 4
    for g in range(W):
        w13 = out[g]["model.layers.1.mlp.experts.w13_weight"]
        assert w13.shape[0] == E // ep
        for j in range(E // ep):
            e = (g % ep) * (E // ep) + j
            gt = O.rne_bf16(full[(f"model.layers.1.mlp.experts.{e}.gate_proj.weight", 1)])
            up = O.rne_bf16(full[(f"model.layers.1.mlp.experts.{e}.up_proj.weight", 1)])
            dn = O.rne_bf16(full[(f"model.layers.1.mlp.experts.{e}.down_proj.weight", 1)])
            assert np.array_equal(w13[j], np.concatenate([gt, up]))
            assert np.array_equal(out[g]["model.layers.1.mlp.experts.w2_weight"][j], dn)


def test_layout_errors():
    with pytest.raises(O.LayoutError):
        _sync("toy", 4, 4, 1, 1)        # kv_heads 2 % TP 4
    with pytest.raises(O.LayoutError):
        _sync("toy-moe", 8, 1, 8, 8)    # 4 experts % EP 8


def _ledger_brute(model, W, tp, dp, ep, rank_map):
    """Per-element: mark each element with its FSDP owner; mark which rollout
    ranks need it (by locating it in the rollout tensors through an index
    tensor pushed through the same sync); count bytes per (owner, dest)."""
    man = manifest(model)
    L = np.zeros((W, W), dtype=np.int64)
    # encode each element's (tensor, flat index) in a uint32 "master" so that
    # its RNE cast is recoverable: use values whose low 16 bits are zero.
    ids = {}
    nxt = 1
    fake = {}
    for k, s in man:
        n = numel(s)
        v = np.arange(nxt, nxt + n, dtype=np.uint32)
        ids[k] = (nxt, s)
        nxt += n
        assert nxt < (1 << 15)
        fake[k] = (v << np.uint32(16)).reshape(s)
    ms = {k: [x[slice(*O.fsdp_rows(x.shape[0], W, r))] for r in range(W)] for k, x in fake.items()}
    out = O.weight_sync(ms, tp, dp, ep, rank_map)
    owner = np.zeros(nxt, dtype=np.int64)
    for k, s in man:
        base, _ = ids[k]
        re = numel(s) // s[0]
        for r in range(W):
            a, b = O.fsdp_rows(s[0], W, r)
            owner[base + a * re: base + b * re] = r
    for g in range(W):
        for x in out[g].values():
            e = x.reshape(-1).astype(np.int64)
            np.add.at(L, (owner[e], g), 2)
    return L


@pytest.mark.parametrize("W,tp,dp,ep", [(2, 2, 1, 1), (4, 2, 2, 2), (8, 2, 4, 4), (3, 1, 3, 1), (8, 1, 8, 1)])
@pytest.mark.parametrize("rank_map", [O.TP_FAST, O.DP_FAST])
def test_ledger_vs_brute_force(W, tp, dp, ep, rank_map):
    for model in ["toy", "toy-moe"] + (["toy-odd"] if tp == 1 else []):
        L = O.ledger(manifest(model), W, tp, dp, ep, rank_map)
        assert np.array_equal(L, _ledger_brute(model, W, tp, dp, ep, rank_map)), model


def test_ledger_real_configs():
    # recv max per GPU (off-diagonal column sums) and totals.
    for model, tp, dp, ep, rmax, tot in (("qwen2.5-7b", 2, 4, 1, 7.33e9, 53.31e9),
                                         ("qwen2.5-32b", 4, 2, 1, 15.71e9, 114.68e9),
                                         ("qwen3-30b-a3b", 2, 4, 8, 7.84e9, 61.61e9)):
        L = O.ledger(manifest(model), 8, tp, dp, ep)
        off = L - np.diag(np.diag(L))
        assert abs(off.sum(axis=0).max() - rmax) / rmax < 0.005
        assert abs(off.sum() - tot) / tot < 0.005
    # R10: the tp-major rank map lowers the 7B recv max to ~5.99 GB
    L = O.ledger(manifest("qwen2.5-7b"), 8, 2, 4, 1, O.DP_FAST)
    off = L - np.diag(np.diag(L))
    assert abs(off.sum(axis=0).max() - 5.99e9) / 5.99e9 < 0.005


def test_transition_ops():
    # SPEC.md:361-363 examples of transition_context.
    assert O.transition_ops(0, 0) == []
    assert O.transition_ops(0, 1) == [(O.OP_OFFLOAD, 0), (O.OP_ONLOAD, 1)]
    assert O.transition_ops(None, 1) == [(O.OP_ONLOAD, 1)]
    assert O.transition_ops(2, 2, True) == [(O.OP_SYNC, 2)]

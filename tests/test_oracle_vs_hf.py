"""Pins the oracle's decoder (oracle/cpu_decoder.py, the fp32 restatement every GPU parity test
compares against) to an independent implementation of the same architectures: HuggingFace
transformers' Llama, Qwen3 and GptOss models, eager attention, fp32, loaded with the oracle's own
weights. The reference (`/root/reference`) has no decoder — its phases are
virtual-time charges (engine.py:251,270,296,358) — so the numerics of the engine-side path are
otherwise pinned only to our own restatement; this test ties that restatement to the standard
definitions (RMSNorm, rotate-half RoPE / YaRN, GQA causal attention, qk-norm, sliding window,
attention sinks, QKV / O biases, SwiGLU, gpt-oss routed experts with the clamped SwiGLU).
CPU only, oracle-sized shapes (the C1 tiny model, Qwen3 and gpt-oss minis)."""

import math

import pytest
import torch

transformers = pytest.importorskip("transformers")

TOL = 1e-5  # fp32 vs fp32, different operation order (measured 0.4-1.2e-6, relative L2 over the logits)


def _prompt(shape, n=24, seed=3):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(3, shape.vocab, (n,), generator=g).tolist()


def _load(model, sd):
    missing, unexpected = model.load_state_dict(sd, strict=False)
    missing = [m for m in missing if "rotary" not in m]
    assert not missing and not unexpected, (missing, unexpected)


def _dense_state(ora, shape):
    s = shape
    H, G, D, F = s.n_q, s.n_kv, s.d_head, s.d_ff
    sd = {"model.embed_tokens.weight": ora.embed, "model.norm.weight": ora.fn, "lm_head.weight": ora.head}
    for i, w in enumerate(ora.layers):
        p = f"model.layers.{i}."
        qkv = w["qkv"]
        sd[p + "input_layernorm.weight"] = w["an"]
        sd[p + "self_attn.q_proj.weight"] = qkv[: H * D]
        sd[p + "self_attn.k_proj.weight"] = qkv[H * D:(H + G) * D]
        sd[p + "self_attn.v_proj.weight"] = qkv[(H + G) * D:]
        sd[p + "self_attn.o_proj.weight"] = w["o"]
        sd[p + "post_attention_layernorm.weight"] = w["mn"]
        if "gu" in w:
            sd[p + "mlp.gate_proj.weight"] = w["gu"][:F]
            sd[p + "mlp.up_proj.weight"] = w["gu"][F:]
            sd[p + "mlp.down_proj.weight"] = w["dn"]
        if "qn" in w:
            sd[p + "self_attn.q_norm.weight"] = w["qn"]
            sd[p + "self_attn.k_norm.weight"] = w["kn"]
        if "bqkv" in w:
            b = w["bqkv"]
            sd[p + "self_attn.q_proj.bias"] = b[: H * D]
            sd[p + "self_attn.k_proj.bias"] = b[H * D:(H + G) * D]
            sd[p + "self_attn.v_proj.bias"] = b[(H + G) * D:]
            sd[p + "self_attn.o_proj.bias"] = w["bo"]
        if "sinks" in w:
            sd[p + "self_attn.sinks"] = w["sinks"]
    return sd


def _compare(model, ora, ids):
    model.eval()
    with torch.no_grad():
        want = model(torch.tensor([ids])).logits[0].float()
    got = ora.forward("r", ids, 0, list(range(len(ids))))
    err = float((got - want).norm() / want.norm())
    assert err < TOL, err
    assert torch.equal(got.argmax(-1), want.argmax(-1))
    return err


@pytest.mark.parametrize("name", ["tiny", "qwen3-mini"])
def test_oracle_matches_hf_dense(name):
    from oracle.cpu_decoder import CpuDecoder
    from paper_2512_15834_b200.modelcfg import QWEN3_MINI, TINY

    shape = {"tiny": TINY, "qwen3-mini": QWEN3_MINI}[name]
    common = dict(vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.d_ff,
                  num_hidden_layers=shape.layers, num_attention_heads=shape.n_q, num_key_value_heads=shape.n_kv,
                  head_dim=shape.d_head, rms_norm_eps=shape.rms_eps, max_position_embeddings=4096,
                  rope_parameters={"rope_type": "default", "rope_theta": shape.rope_theta},
                  tie_word_embeddings=False, attention_bias=False)
    if shape.qk_norm:
        cfg = transformers.Qwen3Config(**common)
        cls = transformers.Qwen3ForCausalLM
    else:
        cfg = transformers.LlamaConfig(mlp_bias=False, **common)
        cls = transformers.LlamaForCausalLM
    cfg._attn_implementation = "eager"
    model = cls(cfg).float()
    ora = CpuDecoder(shape)
    _load(model, _dense_state(ora, shape))
    _compare(model, ora, _prompt(shape))


def test_oracle_matches_hf_gpt_oss():
    """gpt-oss mini (C4 family): biases, sinks, a 32-token sliding window on layer 0 (a 48-token
    prompt exercises it), YaRN, 16 MXFP4 experts top-4 (the oracle's dequantised weights)."""
    from oracle.cpu_decoder import CpuDecoder
    from paper_2512_15834_b200.modelcfg import GPT_OSS_MINI

    s = GPT_OSS_MINI
    factor, bfast, bslow, orig = s.yarn
    cfg = transformers.GptOssConfig(
        vocab_size=s.vocab, hidden_size=s.d_model, intermediate_size=s.d_ff, num_hidden_layers=s.layers,
        num_attention_heads=s.n_q, num_key_value_heads=s.n_kv, head_dim=s.d_head, rms_norm_eps=s.rms_eps,
        num_local_experts=s.n_experts, num_experts_per_tok=s.top_k, sliding_window=s.sliding_window,
        swiglu_limit=s.swiglu_limit, attention_bias=True, tie_word_embeddings=False,
        max_position_embeddings=131072,
        layer_types=["sliding_attention" if s.window(i) else "full_attention" for i in range(s.layers)],
        rope_parameters={"rope_type": "yarn", "factor": factor, "beta_fast": bfast, "beta_slow": bslow,
                         "truncate": False, "original_max_position_embeddings": orig, "rope_theta": s.rope_theta})
    cfg._attn_implementation = "eager"
    model = transformers.GptOssForCausalLM(cfg).float()
    ora = CpuDecoder(s)
    sd = _dense_state(ora, s)
    for i, w in enumerate(ora.layers):
        p = f"model.layers.{i}.mlp."
        sd[p + "router.weight"] = w["router"]
        sd[p + "router.bias"] = w["router_b"]
        ex = [w["expert"](e) for e in range(s.n_experts)]  # (w_gate_up [2F][d], b, w_down [d][F], b)
        sd[p + "experts.gate_up_proj"] = torch.stack([e[0].T for e in ex])
        sd[p + "experts.gate_up_proj_bias"] = torch.stack([e[1] for e in ex])
        sd[p + "experts.down_proj"] = torch.stack([e[2].T for e in ex])
        sd[p + "experts.down_proj_bias"] = torch.stack([e[3] for e in ex])
    _load(model, sd)
    _compare(model, ora, _prompt(s, n=48))
    assert math.isfinite(float(ora.head.sum()))

"""Numerics parity at the BASELINE widths: full-width 2-layer slices of
Llama-2-7B (C2), Llama-2-70B (C3/C4: GQA 64/8) and BLOOM-176B (C5: d=14336,
V=250880, ALiBi) run through ModelRunner (tcgen05 prefill of a 1024-token
prompt writing the paged pool, then CUDA-graph decode steps) and through the
fp32 CPU oracle (oracle/decoder.py) on the same random-init weights.

Checked per config: teacher-forced logits (the oracle is fed the GPU's
tokens) within the stated bf16-vs-fp32 tolerance, and greedy agreement —
the GPU's token equals the oracle's argmax at every checked step whose
oracle top-2 margin exceeds twice that step's observed logit error (such a
step cannot flip by rounding; closer margins are counted as near-ties and
reported, not asserted).  ``greedy_horizon`` is the number of leading steps
on which the tokens agree.  Beside the fp32 oracle runs its bf16-storage twin
(OracleDecoder(emulate_bf16=True): the same fp32 math with every activation
the device stores in bf16 rounded there); its distance to the fp32 oracle is
the error bf16 storage alone explains, reported as ``emul_dlogit``.
Observed errors are written to gpurun_out/parity_widths.json.

Tolerances: max |logit_gpu - logit_oracle| over all checked steps <=
TOL_REL[model] * max |logit|, TOL_REL = 3x the relative error observed on
B200 (profiles/r2_parity_widths.json: 0.48 % / 2.2 % / 0.69 %), rounded up;
and <= EMUL_FACTOR x the bf16-storage twin's error (observed ratio 1.04-1.11:
the kernels add almost nothing on top of storing activations in bf16).
"""

import dataclasses
import json
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

P, N_OUT = 1024, 16
# model -> max |dlogit| / max |logit| allowed (3x observed, see module docstring)
TOL_REL = {"llama2-7b": 0.015, "llama2-70b": 0.07, "bloom-176b": 0.021}
EMUL_FACTOR = 1.5


def _record(name, rec):
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    p = os.path.join(d, "parity_widths.json")
    try:
        with open(p) as f:
            allr = json.load(f)
    except Exception:
        allr = {}
    allr[name] = rec
    with open(p, "w") as f:
        json.dump(allr, f, indent=1)


def run_slice(model, layers=2, prompt_len=P, n_out=N_OUT, seed=0):
    from paper_2311_18677_b200 import kernels as K
    from paper_2311_18677_b200.kvcache import KVCacheManager
    from paper_2311_18677_b200.model import get_config, init_weights
    from paper_2311_18677_b200.runner import ModelRunner
    cfg = dataclasses.replace(get_config(model), n_layers=layers, name=f"{model}-{layers}L")
    w = init_weights(cfg, seed=seed)
    nb = (prompt_len + n_out + 15) // 16 + 4
    kv = KVCacheManager(layers, nb, cfg.n_kv_heads, cfg.head_dim, 16, 2, nb)
    runner = ModelRunner(w, kv)
    prompt = torch.randint(0, cfg.vocab, (prompt_len,),
                           generator=torch.Generator().manual_seed(seed + 11)).tolist()
    seq = kv.allocate(prompt_len + n_out)
    toks = torch.tensor(prompt, dtype=torch.int32, device="cuda")
    slots = torch.empty(prompt_len, dtype=torch.int32, device="cuda")
    K.slots_from_table(kv.table_row_ptr(seq), 0, prompt_len, 16, slots)
    first = runner.prefill(toks, [prompt_len], ModelRunner.pack_meta([prompt_len]).cuda(),
                           local_slots=slots)
    logits = [runner.plogits[0].clone()]
    g = runner.decode_graph(1, prompt_len + n_out, n_out)
    g.load([seq], first[:1], [prompt_len])
    g.capture()
    for _ in range(n_out - 1):
        g.replay()
        logits.append(g.logits[0].clone())
    torch.cuda.synchronize()
    gpu_toks = [int(first[0])] + g.out_ring[0, :n_out - 1].tolist()
    gpu_logits = torch.stack(logits).cpu()
    from oracle.decoder import OracleDecoder
    orc = OracleDecoder.from_weights(w)
    del runner, g, kv
    torch.cuda.empty_cache()
    ref_toks, ref_logits = orc.generate(prompt, n_out, forced=gpu_toks[:-1])
    twin = OracleDecoder(cfg, orc.layers, orc.embed, orc.lm_head, orc.final_norm,
                         extra=orc.extra, emulate_bf16=True)
    _, emul_logits = twin.generate(prompt, n_out, forced=gpu_toks[:-1])
    return cfg, gpu_toks, gpu_logits, ref_toks, ref_logits, emul_logits


def compare(gpu_toks, gpu_logits, ref_toks, ref_logits, tol_rel, emul_logits=None):
    tol = tol_rel * float(ref_logits.abs().max())
    diff = (gpu_logits - ref_logits).abs().max(-1).values
    top2 = ref_logits.topk(2, -1).values
    margin = top2[:, 0] - top2[:, 1]
    agree = [a == b for a, b in zip(gpu_toks, ref_toks)]
    decisive = (margin > 2 * diff).tolist()
    horizon = 0
    for a in agree:
        if not a:
            break
        horizon += 1
    emul = (None if emul_logits is None else
            float((emul_logits - ref_logits).abs().max(-1).values.max()))
    return {"max_dlogit": float(diff.max()), "mean_dlogit": float(diff.mean()),
            "emul_dlogit": emul, "max_logit": float(ref_logits.abs().max()), "tol": tol,
            "tol_rel": tol_rel, "rel_dlogit": float(diff.max()) / float(ref_logits.abs().max()),
            "greedy_horizon": horizon, "steps": len(agree),
            "agree": sum(agree), "near_ties": int(sum(1 for d in decisive if not d)),
            "disagree_decisive": int(sum(1 for a, d in zip(agree, decisive) if d and not a))}


@pytest.mark.parametrize("model", ["llama2-7b", "llama2-70b", "bloom-176b"])
def test_full_width_slice_matches_oracle(model):
    cfg, gt, gl, rt, rl, el = run_slice(model)
    rec = compare(gt, gl, rt, rl, TOL_REL[model], el)
    rec.update({"model": cfg.name, "prompt": P, "n_out": N_OUT, "d_model": cfg.d_model,
                "n_heads": cfg.n_heads, "n_kv_heads": cfg.n_kv_heads, "vocab": cfg.vocab})
    _record(model, rec)
    print(json.dumps(rec))
    assert rec["max_dlogit"] <= rec["tol"], rec
    assert rec["max_dlogit"] <= EMUL_FACTOR * rec["emul_dlogit"], rec
    assert rec["disagree_decisive"] == 0, rec

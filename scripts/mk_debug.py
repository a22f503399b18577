"""Diagnose per-step vs persistent forward differences at the 64-token verify shape.

Checks, on identical staged inputs: each path run twice (determinism), and each path
with the batch split into 4 x 16-token launches (batch invariance: must be identical)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import test_gpu_mk as M
from paper_2410_11305_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "7b2l"
model = M.model_of(name)
eng = M._engine(model, 16)
B, G1, cfg = 16, eng.gamma + 1, eng.cfg
committed = eng.t["committed"].clone()
g = torch.Generator(device="cuda").manual_seed(1)
toks = torch.randint(0, cfg.vocab_size, (B * G1,), dtype=torch.int32, device="cuda", generator=g)
pos = (committed.repeat_interleave(G1) + torch.arange(G1, device="cuda").repeat(B)).int()
eng.t["tok"][:B * G1].copy_(toks)
eng.t["pos"][:B * G1].copy_(pos)
eng.t["slot"][:B * G1].copy_(torch.arange(B, device="cuda").repeat_interleave(G1).int())
big = eng.verify_batches
eng2 = eng
# split descriptor: 4 batches of 4 sequences (16 tokens)
import paper_2410_11305_b200.engine as E
save_B = eng.B
small = []
for s0 in range(0, B, 4):
    tok0 = torch.tensor([i * G1 for i in range(4)], dtype=torch.int32, device="cuda")
    ntok = torch.full((4,), G1, dtype=torch.int32, device="cuda")
    eng._blk[("dbg", s0)] = (tok0, ntok)
    off = s0 * G1 * 4
    b = _lib.Batch(T=4 * G1, tokens=eng.t["tok"].data_ptr() + off, positions=eng.t["pos"].data_ptr() + off,
                   slots=eng.t["slot"].data_ptr() + off, n_blk=4, blk_tok0=tok0.data_ptr(), blk_ntok=ntok.data_ptr(),
                   blk_qmax=G1, ctx_cap=eng.kv.capacity)
    small.append((b, off))
st = _lib.stream_ptr()


def run(fn, batches):
    logits = torch.full((64, cfg.vocab_size), float("nan"), device="cuda")
    arg = torch.full((64,), -1, dtype=torch.int32, device="cuda")
    for b, off in batches:
        _lib.call(fn, eng.cm, b, _lib.QS_MODE_HIGH, eng.ws, logits[off // 4:].data_ptr(), arg.data_ptr() + off, st)
    torch.cuda.synchronize()
    return logits.clone(), [k.clone() for k in eng.kv.k]


res = {}
for fn in ("qs_forward", "qs_forward_mk"):
    for nm, bt in (("T64", big), ("4xT16", small)):
        for rep in range(2):
            res[(fn, nm, rep)] = run(fn, bt)
base = res[("qs_forward", "4xT16", 0)]
for k, (lg, kk) in res.items():
    print(k, "logit diff vs per-step 4xT16:", float((lg - base[0]).abs().max()),
          "K0 diff", float((kk[0] - base[1][0]).abs().max()))

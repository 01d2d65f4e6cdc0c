#!/usr/bin/env python
"""Regenerate the golden fixtures from the UNMODIFIED reference (oracle/_ref/libsafekv_ref.so,
built from /root/reference/proj/include).  Run here (the reference is not on the GPU box):

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed):
  cfg1_workload.npz   config 1 = safekv::generate(WorkloadSpec{SingleRequestPII, n_users=4,
                      n_requests=1000, inter=0.05, intra=0.0, secret_density=0.3, ctx=0, seed=2})
                      (workload.hpp:428-700; values from presets/single_request_pii.json), with the
                      reference canonical_bytes() FNV digest
  cfg1_expected.npz   Appendix-A outputs of the reference for config 1 (B=16, W=32): batch 1 on an
                      empty index, commit, epoch, batch 2 = the same prompts again (warm index),
                      commit, epoch -- hashes, masks, labels, decisions, match lengths, tiers,
                      events, final index export
  scan_kats.json      reference verdicts (sensitive, categories, per-rule mask) for the reference's
                      own known-answer strings (test_detection.cpp:33-77, :110-118) and the
                      generate_rule_corpus(500, 77) corpus (test_workload.cpp:209-218)
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from refh import RefEngine, RefRules, load_ref, reference_workload  # noqa: E402

KAT_TEXTS = [
    "my ssn is 123-45-6789", "the weather is nice", "status of PROJECT-TITAN today", "see (PROJECT-TITAN).",
    "PROJECT-TITANIC is something else", "my ssn is 987-65-4321", "call me at (415) 555-0134",
    "email me at user99@mail01.com", "server at 10.4.77.3", "card number 4111-1111-1111-1111",
    "account number 48392057", "device mac 0a:1b:2c:3d:4e:5f", "imei 490154203237518", "danger zone",
    "x123-45-6789", "123-45-67890", "((PROJECT-TITAN))", ".PROJECT-TITAN.x", "account no.123456",
    "account\tnumber  1234567", "imei490154203237518", "10.0.0.1.", "a@b.c", "a@b.cd",
]


def to_tokens(texts):
    offs = np.zeros(len(texts) + 1, np.uint64)
    for i, t in enumerate(texts):
        offs[i + 1] = offs[i] + len(t)
    tok = np.frombuffer(b"".join(texts), np.uint8).astype(np.uint32)
    return tok, offs


def main():
    L = load_ref()
    assert L is not None, "build the reference harness first: make -C oracle ref"
    texts, users, owners, truth, digest = reference_workload(L, 0, 4, 1000, 0.05, 0.0, 0.3, 0.0, 2)
    tok, offs = to_tokens(texts)
    tb, te, ts, tcount = [], [], [], []
    for spans in truth:
        tcount.append(len(spans))
        for b, e, s in spans:
            tb.append(b)
            te.append(e)
            ts.append(s)
    np.savez_compressed(HERE / "cfg1_workload.npz", tokens=tok.astype(np.uint8), offsets=offs,
                        users=np.array(users, np.uint64), owners=np.array(owners, np.uint8),
                        truth_count=np.array(tcount, np.uint32), truth_begin=np.array(tb, np.uint64),
                        truth_end=np.array(te, np.uint64), truth_sens=np.array(ts, np.uint8),
                        digest=np.array([digest], np.uint64))
    rules = RefRules(L)
    eng = RefEngine(L, rules, B=16, W=32)
    out = {}
    for rnd in (1, 2):
        o = eng.admit(tok, offs, np.array(users, np.uint64), np.array(owners, np.uint8))
        for k, v in o.items():
            out[f"r{rnd}_{k}"] = v
        eng.commit()
        ep, ev = eng.epoch()
        out[f"r{rnd}_epoch"] = np.array([ep], np.uint64)
        out[f"r{rnd}_events"] = np.array([(e[0], e[1], e[2], e[5]) for e in ev], np.uint64).reshape(-1, 4)
    x = eng.export()
    for k, v in x.items():
        out[f"export_{k}"] = v
    np.savez_compressed(HERE / "cfg1_expected.npz", **out)
    eng.close()

    kats = []
    for t in KAT_TEXTS:
        b = t.encode()
        s, cats = rules.verdict(b)
        kats.append({"text": t, "sensitive": s, "categories": cats, "mask": rules.mask(b)})
    # generate_rule_corpus(500, 77): every text is flagged (test_workload.cpp:209-218)
    import ctypes as C
    lens = np.zeros(500, np.uint32)
    total = L.ref_rule_corpus(500, 77, None, 0, lens.ctypes.data)
    buf = C.create_string_buffer(total)
    L.ref_rule_corpus(500, 77, buf, total, lens.ctypes.data)
    pos = 0
    corpus = []
    for n in lens.tolist():
        raw = buf.raw[pos:pos + n]
        pos += n
        s, cats = rules.verdict(raw)
        corpus.append({"text": raw.decode("latin-1"), "sensitive": s, "categories": cats, "mask": rules.mask(raw)})
    (HERE / "scan_kats.json").write_text(json.dumps({"kats": kats, "rule_corpus_500_77": corpus}, indent=1))
    print("cfg1 digest %016x, %d blocks" % (digest, len(out["r1_block_h"])))


if __name__ == "__main__":
    main()

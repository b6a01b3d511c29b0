"""Toy worked-example (cfg1) input builders shared by oracle and GPU tests (no method arithmetic)."""
import numpy as np

from inputs import synth


def toy_pool(toy, T):
    V = toy["V"]
    rows = {name: synth.logits_from_probs(V, {int(t): p for t, p in spec.items()})
            for name, spec in toy["rows"].items()}
    pool = np.stack([rows[toy["node_rows"][min(i, len(toy["node_rows"]) - 1)]] for i in range(T)])
    return pool[None].astype(np.float32)


def toy_target(toy, T, tok_fill=0):
    V = toy["V"]
    tg = np.zeros((1, T, V), np.float32)
    for node, t in toy["verify"]["argmax"].items():
        tg[0, int(node), t] = 5.0
    for i in range(T):
        if str(i) not in toy["verify"]["argmax"]:
            tg[0, i, 31] = 5.0  # a token that is never drafted
    return tg

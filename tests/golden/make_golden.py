"""Generate the golden vectors that pin the oracle (and, through it, the CUDA path).

Runs the REFERENCE package (``ringmpc`` from /root/reference/pkg/src) -- never
this repo's code -- and writes ``tests/golden/golden.npz`` plus
``tests/golden/golden.json``.  It only runs in the build container (the
reference does not exist on the GPU box); the outputs are committed.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Case recipes mirror the reference's own tests so the inputs can be regenerated
bit-for-bit by numpy alone (see tests/golden_cases.py):

* relu/drelu per-party shares + per-round payload digests + meter traces for
  the Fig. 4 example, the 10k agreement case (test_simulator.py:70-88),
  Theorem-1/2 exhaustive sweeps (test_acceptance.py:31-94), odd sizes from
  test_protocol.py:372-418 and the BASELINE windows at n=4096;
* stage kernels: beaver_mul/beaver_and/circuit_add/a2b/b2a_bit
  (test_protocol.py:110-271);
* pack layouts for w = 1..64 (test_transport.py:22-48);
* dealer streams and the HBTRIP1 golden SHA (test_dealer.py:14,82-86);
* the simulator: sim_relu outputs, sim_forward / plain_forward logits, DReLU masks and
  activation ranges on the desk models (simulator.py:33-174).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for golden_cases

from ringmpc import dealer, protocol, ring, sharing, transport  # noqa: E402  (reference package)
from ringmpc.protocol import ProtocolSession  # noqa: E402
from ringmpc.ring import BitWindow, FixedPointConfig  # noqa: E402

import golden_cases as gc  # noqa: E402


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


class RecordingEndpoint(transport.LocalEndpoint):
    def __init__(self, *a):
        super().__init__(*a)
        self.sent: list[bytes] = []

    def exchange(self, payload: bytes) -> bytes:
        self.sent.append(bytes(payload))
        return super().exchange(payload)


def rec_pair():
    import queue

    q01, q10 = queue.Queue(), queue.Queue()
    return RecordingEndpoint(0, q10, q01), RecordingEndpoint(1, q01, q10)


def sessions(bool_width=0, bool_count=0, arith_width=0, arith_count=0, seed=0):
    """Same stocking as the reference tests/conftest.py:26-47, with recording endpoints."""
    ep0, ep1 = rec_pair()
    batches = []
    if bool_count:
        batches.append(dealer.gen_bool_triples(bool_count, bool_width, seed=seed * 2 + 1))
    if arith_count:
        batches.append(dealer.gen_arith_triples(arith_count, arith_width, seed=seed * 2 + 2))
    out = []
    for party, ep in ((0, ep0), (1, ep1)):
        st = dealer.TripleStore(party)
        for b in batches:
            st.add_batch(b)
        out.append(ProtocolSession(ep, st, FixedPointConfig()))
    return out[0], out[1], (ep0, ep1)


def relu_sessions(count, w, n_bits, seed):
    need = protocol.relu_triple_cost(count, w, n_bits)
    return sessions(w, need[(dealer.BOOL, w)], n_bits, need[(dealer.ARITH, n_bits)], seed)


ARR: dict[str, np.ndarray] = {}
META: dict[str, dict] = {}


def record(name, r0, r1, eps, keep_arrays, extra=None):
    y0 = np.asarray(r0.data, dtype=np.uint64).reshape(-1)
    y1 = np.asarray(r1.data, dtype=np.uint64).reshape(-1)
    meta = {
        "y0_sha": sha(y0),
        "y1_sha": sha(y1),
        "trace0": [list(t) for t in eps[0].meter.trace],
        "trace1": [list(t) for t in eps[1].meter.trace],
        "payload0_sha": [sha(p) for p in eps[0].sent],
        "payload1_sha": [sha(p) for p in eps[1].sent],
    }
    if extra:
        meta.update(extra)
    if keep_arrays:
        ARR[name + "/y0"] = y0
        ARR[name + "/y1"] = y1
    META[name] = meta


def relu_case(name, op, x0, x1, n_bits, k, m, seed, keep_arrays):
    win = BitWindow(k, m)
    s0, s1, eps = relu_sessions(x0.size, win.width, n_bits, seed)
    t0 = sharing.ArithShareTensor(0, n_bits, x0)
    t1 = sharing.ArithShareTensor(1, n_bits, x1)
    fn = protocol.relu if op == "relu" else protocol.drelu
    r0, r1 = transport.run_parties(lambda: fn(s0, t0, win), lambda: fn(s1, t1, win), endpoints=eps)
    rec = sharing.reconstruct_arith(r0, r1)
    record(name, r0, r1, eps, keep_arrays, {"op": op, "n_bits": n_bits, "k": k, "m": m, "seed": seed,
                                              "n": int(x0.size), "recon_sha": sha(rec)})
    if keep_arrays:
        ARR[name + "/recon"] = rec
    return rec


def main():
    # ---------------- ReLU / DReLU cases (recipes in golden_cases.RELU_CASES)
    for case in gc.RELU_CASES:
        x0, x1 = gc.make_inputs(case)
        rec = relu_case(case["name"], case["op"], x0, x1, case["n_bits"], case["k"], case["m"],
                        case["seed"], case.get("keep", False))
        if case.get("store_inputs"):
            ARR[case["name"] + "/x0"] = x0
            ARR[case["name"] + "/x1"] = x1
        if case["name"] == "sim10k_21_7":
            # protocol == simulator on the same split (test_simulator.py:70-88)
            from ringmpc.simulator import drelu_from_shares

            keep = drelu_from_shares(x0, x1, 64, BitWindow(21, 7))
            assert np.array_equal(rec, ring.mul_mod((x0 + x1) & np.uint64(2**64 - 1), keep, 64))

    # ---------------- stage kernels
    for case in gc.STAGE_CASES:
        ins = gc.make_stage_inputs(case)
        kind = case["op"]
        if kind == "beaver_mul":
            w = case["w"]
            s0, s1, eps = sessions(arith_width=w, arith_count=ins["x0"].size, seed=case["seed"])
            A = [sharing.ArithShareTensor(p, w, ins[f"x{p}"]) for p in (0, 1)]
            B = [sharing.ArithShareTensor(p, w, ins[f"y{p}"]) for p in (0, 1)]
            r0, r1 = transport.run_parties(lambda: protocol.beaver_mul(s0, A[0], B[0]),
                                           lambda: protocol.beaver_mul(s1, A[1], B[1]), endpoints=eps)
        elif kind in ("beaver_and", "circuit_add"):
            w = case["w"]
            cnt = ins["x0"].size * (1 if kind == "beaver_and" else 1 + 2 * protocol.prefix_levels(w))
            s0, s1, eps = sessions(bool_width=w, bool_count=cnt, seed=case["seed"])
            A = [sharing.BinShareTensor(p, w, ins[f"x{p}"]) for p in (0, 1)]
            B = [sharing.BinShareTensor(p, w, ins[f"y{p}"]) for p in (0, 1)]
            fn = protocol.beaver_and if kind == "beaver_and" else protocol.circuit_add
            r0, r1 = transport.run_parties(lambda: fn(s0, A[0], B[0]), lambda: fn(s1, A[1], B[1]), endpoints=eps)
        elif kind == "a2b":
            w = case["w"]
            s0, s1, eps = sessions(bool_width=w, bool_count=ins["x0"].size * (1 + 2 * protocol.prefix_levels(w)),
                                   seed=case["seed"])
            A = [sharing.ArithShareTensor(p, w, ins[f"x{p}"]) for p in (0, 1)]
            r0, r1 = transport.run_parties(lambda: protocol.a2b(s0, A[0]), lambda: protocol.a2b(s1, A[1]),
                                           endpoints=eps)
        elif kind == "b2a":
            nb = case["n_bits"]
            s0, s1, eps = sessions(arith_width=nb, arith_count=ins["x0"].size, seed=case["seed"])
            A = [sharing.BinShareTensor(p, 1, ins[f"x{p}"]) for p in (0, 1)]
            r0, r1 = transport.run_parties(lambda: protocol.b2a_bit(s0, A[0], nb),
                                           lambda: protocol.b2a_bit(s1, A[1], nb), endpoints=eps)
        else:
            raise ValueError(kind)
        record(case["name"], r0, r1, eps, case.get("keep", False), {"op": kind})

    # ---------------- packing layouts (test_transport.py:22-48)
    rng = np.random.default_rng(1)
    blobs, offs, counts = [], [0], []
    for w in range(1, 65):
        n = int(rng.integers(1, 200))
        vals = np.frombuffer(rng.bytes(8 * n), dtype="<u8").copy() & np.uint64((1 << w) - 1)
        blob = transport.pack_words(vals, w)
        assert len(blob) == transport.packed_nbytes(n, w)
        blobs.append(np.frombuffer(blob, dtype=np.uint8))
        offs.append(offs[-1] + len(blob))
        counts.append(n)
    ARR["pack/blob"] = np.concatenate(blobs)
    ARR["pack/offsets"] = np.array(offs, dtype=np.int64)
    ARR["pack/counts"] = np.array(counts, dtype=np.int64)

    # ---------------- dealer streams
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "g.bin")
        dealer.save_triples(dealer.gen_arith_triples(1000, 16, seed=1234), p)
        META["dealer_hbtrip1_sha"] = {"sha": hashlib.sha256(open(p, "rb").read()).hexdigest()}
    dl = {}
    for kind, cnt, w, seed in (("arith", 777, 64, 9), ("bool", 1000, 8, 3), ("bool", 513, 6, 11), ("arith", 100, 10, 5)):
        gen = dealer.gen_arith_triples if kind == "arith" else dealer.gen_bool_triples
        b = gen(cnt, w, seed)
        dl[f"{kind}_{w}_{seed}_{cnt}"] = [sha(a) for p_ in (0, 1) for a in b.party_arrays(p_)]
    META["dealer_streams"] = dl

    # ---------------- ring linear layers (nn.py:198-259), per party
    from ringmpc import models, nn
    from ringmpc.cli import run_local_forward

    class _Sess:  # the layer functions only read session.fxp
        fxp = FixedPointConfig(64, 16)

    for case in gc.NN_CASES:
        ins = gc.make_nn_inputs(case)
        outs = []
        for party in (0, 1):
            x = sharing.ArithShareTensor(party, 64, ins[f"x{party}"])
            if case["op"] == "linear":
                r = nn.linear_forward(_Sess, x, ins["w"], ins["b"])
            elif case["op"] == "conv":
                r = nn.conv2d_forward(_Sess, x, nn.Conv2d(*case["layer"], weight="w", bias="b"), ins["w"], ins["b"])
            elif case["op"] == "avgpool":
                r = nn.avgpool_forward(_Sess, x, nn.AvgPool(*case["layer"]))
            else:
                r = nn.truncate_local(x, _Sess.fxp)
            outs.append(np.asarray(r.data, dtype=np.uint64))
        META[case["name"]] = {"y0_sha": sha(outs[0]), "y1_sha": sha(outs[1]), "shape": list(outs[0].shape)}

    # ---------------- model-level entry: run_local_forward (cli.py:159-180) on desk models
    for mc in gc.MODEL_CASES:
        model = models.build_cnn(11) if mc["arch"] == "cnn" else models.build_mlp(11)
        for name, arr in model.weights.items():
            ARR[f"model_{mc['arch']}/{name}"] = arr
        x_f = gc.model_inputs(mc)
        cfg = nn.ReluConfig([None if w is None else BitWindow(*w) for w in mc["windows"]])
        logits, meters, logs, _ = run_local_forward(model, cfg, x_f, mc["seed"])
        META[mc["name"]] = {"logits_sha": sha(np.ascontiguousarray(logits).view(np.uint64)),
                            "meter0": meters[0].to_json(), "meter1": meters[1].to_json(),
                            "layers0": logs[0], "layers1": logs[1]}
        ARR[mc["name"] + "/logits"] = logits

    # ---------------- simulator (simulator.py:33-174): sim_relu, sim_forward, plain_forward, ranges
    from ringmpc import simulator as sim

    for case in gc.SIM_RELU_CASES:
        x = gc.sim_relu_input(case)
        rng = np.random.default_rng(np.random.SeedSequence(case["split_seed"]))
        out = sim.sim_relu(x, BitWindow(case["k"], case["m"]), FixedPointConfig(64, 16), rng)
        ARR[case["name"] + "/out"] = out
        META[case["name"]] = {"out_sha": sha(np.ascontiguousarray(out).view(np.uint64))}
    for mc in gc.SIM_MODEL_CASES:
        model = models.build_cnn(11) if mc["arch"] == "cnn" else models.build_mlp(11)
        x_f, labels = gc.sim_model_inputs(mc)
        cfg = sim.SimConfig(FixedPointConfig(64, 16), [None if w is None else BitWindow(*w) for w in mc["windows"]],
                            seed=mc["seed"])
        logits, acc = sim.sim_forward(model, x_f, labels, cfg)
        _, masks = sim.collect_drelu_decisions(model, x_f, cfg)
        ARR[mc["name"] + "/logits"] = logits
        ARR[mc["name"] + "/plain"] = sim.plain_forward(model, x_f)
        for i, mk in enumerate(masks):
            ARR[mc["name"] + f"/mask{i}"] = mk
        META[mc["name"]] = {"accuracy": acc, "n_masks": len(masks),
                            "ranges": {str(g): v for g, v in sim.collect_activation_ranges(model, x_f).items()}}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **ARR)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(META, fh, indent=1, sort_keys=True)
    print(f"wrote {len(ARR)} arrays, {len(META)} cases")


if __name__ == "__main__":
    main()

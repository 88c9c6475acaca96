"""Diagnostics: 3xTF32 accuracy vs K / split-K chunking; slice-sum check."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

MODE = sys.argv[1] if len(sys.argv) > 1 else "all"


def tc_err(m, n, k, seed=0, positive=False):
    import torch
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn((m, k), dtype=torch.complex64, device="cuda", generator=g)
    b = torch.randn((k, n), dtype=torch.complex64, device="cuda", generator=g)
    if positive:
        a = a.real.abs().to(torch.complex64)
        b = b.real.abs().to(torch.complex64)
    A = DenseTensor([Index("m", m), Index("k", k)], a)
    B = DenseTensor([Index("k", k), Index("n", n)], b)
    got = contract_pair(A, B, variant=int(os.environ.get("TNC_VARIANT", "4"))).data.to(torch.complex128)
    simt = contract_pair(A, B, variant=1).data.to(torch.complex128)
    want = a.to(torch.complex128) @ b.to(torch.complex128)
    return ((got - want).norm() / want.norm()).item(), ((simt - want).norm() / want.norm()).item()


if MODE in ("all", "prec"):
    for split in ("1", "4", "16"):
        for k in (256, 1024, 4096, 16384):
            out = subprocess.run([sys.executable, __file__, "one", "256", "256", str(k)], env=dict(os.environ, TNC_KSPLIT=split),
                                 capture_output=True, text=True)
            print(f"split={split} K={k}: {out.stdout.strip()} {out.stderr.strip()[-300:]}", flush=True)
    out = subprocess.run([sys.executable, __file__, "pos", "256", "256", "4096"], env=dict(os.environ, TNC_KSPLIT="1"),
                         capture_output=True, text=True)
    print("positive K=4096:", out.stdout.strip(), out.stderr.strip()[-300:])
if MODE == "one":
    print("tc %.3e simt %.3e" % tc_err(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])))
if MODE == "pos":
    print("tc %.3e simt %.3e" % tc_err(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), positive=True))
if MODE in ("all", "slices"):
    import itertools
    import numpy as np
    from conftest import arr, load_golden, rel_l2
    from paper_2504_09186_b200 import SliceSpec, circuit_to_network, greedy_path, linearize, parse_circuit, permute
    from paper_2504_09186_b200.execute import SliceExecutor
    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=g["open"])
    t = greedy_path(net, 0)
    spec = SliceSpec.from_json(json.dumps(g["open_net"]["slice_spec"]))
    ex = SliceExecutor(net, linearize(t), spec, "single")
    bad = []
    for sid, item in enumerate(g["open_net"]["per_slice"]):
        root = ex.run_slice(spec.assignment(sid))
        by = {ix.label: ix for ix in root.indices}
        got = permute(root, [by[l] for l in item["labels"]]).numpy()
        e = rel_l2(got, arr(item["data"]))
        if not e <= 1e-5:
            bad.append((sid, e))
    print("bad slices", len(bad), bad[:10])
    total = ex.run(range(spec.n_subtasks))
    by = {ix.label: ix for ix in total.indices}
    labels0 = g["open_net"]["per_slice"][0]["labels"]
    want = sum(arr(it["data"]).astype(np.complex128) for it in g["open_net"]["per_slice"])
    got = permute(total, [by[l] for l in labels0]).numpy()
    print("total err", rel_l2(got, want), got[:3], want[:3])

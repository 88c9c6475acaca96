"""Independent complex128 device checker (TEST INFRASTRUCTURE ONLY).

Re-runs a contraction schedule on the GPU with plain torch complex128 ops --
an offset-table gather for every operand permutation and one cuBLAS zgemm per
step -- following the reference semantics directly:

* ``project`` fixes sliced labels (reference ``tensor.py:277-292``);
* ``contract`` sums over the shared labels and returns legs
  free_A ++ free_B in operand order (reference ``contract.py:58-75,149-165``);
* the step loop consumes SSA values exactly once (reference
  ``execute.py:119-178``).

None of the engine's planners, kernels or index maps are used, so agreement
with the engine is evidence at sizes the numpy oracle cannot reach (full C3
slices, C4 sub-slices, the rank-30 C2 chain).  The checker itself is pinned
to the numpy oracle / reference goldens on small cases in
``tests/test_gpu_devcheck.py``.
"""

from __future__ import annotations

import torch

CHUNK = 1 << 24  # gather output elements per offset chunk


def _strides(dims):
    out, step = [], 1
    for d in reversed(dims):
        out.append(step)
        step *= d
    return out[::-1]


def _offsets(dims_of, stride_of, order, device):
    off = torch.zeros(1, dtype=torch.int64, device=device)
    for l in order:
        off = (off[:, None] + torch.arange(dims_of[l], device=device, dtype=torch.int64)[None, :]
               * stride_of[l]).reshape(-1)
    return off


def permute(t, target):
    """t = (labels, dims, flat tensor) -> same tensor in ``target`` order
    (offset-table gather in chunks: high legs x low legs)."""
    labels, dims, data = t
    target = list(target)
    if list(labels) == target:
        return t
    dim_of = dict(zip(labels, dims))
    stride_of = dict(zip(labels, _strides(dims)))
    # split target legs so the low table has at most CHUNK entries
    n_low, size = 0, 1
    for l in reversed(target):
        if size * dim_of[l] > CHUNK:
            break
        size *= dim_of[l]
        n_low += 1
    hi_legs, lo_legs = target[: len(target) - n_low], target[len(target) - n_low:]
    lo = _offsets(dim_of, stride_of, lo_legs, data.device)
    hi = _offsets(dim_of, stride_of, hi_legs, data.device)
    out = torch.empty_like(data)
    nl = lo.numel()
    rows = max(1, CHUNK // nl)
    for r0 in range(0, hi.numel(), rows):
        h = hi[r0:r0 + rows]
        out[r0 * nl:(r0 + h.numel()) * nl] = data[(h[:, None] + lo[None, :]).reshape(-1)]
    return (tuple(target), tuple(dim_of[l] for l in target), out)


def project(t, assignment):
    labels, dims, data = t
    if not any(l in assignment for l in labels):
        return t
    sel = tuple(assignment[l] if l in assignment else slice(None) for l in labels)
    kept = [(l, d) for l, d in zip(labels, dims) if l not in assignment]
    arr = data.reshape(tuple(dims))[sel].reshape(-1).clone() if dims else data.clone()
    return (tuple(l for l, _ in kept), tuple(d for _, d in kept), arr)


def contract(a, b):
    """Sum over shared labels; output legs free_A ++ free_B."""
    la, da, xa = a
    lb, db, xb = b
    sb = set(lb)
    common = [l for l in la if l in sb]
    cs = set(common)
    fa = [l for l in la if l not in cs]
    fb = [l for l in lb if l not in cs]
    dim = dict(zip(la, da))
    dim.update(zip(lb, db))
    for l in common:
        if dict(zip(la, da))[l] != dict(zip(lb, db))[l]:
            raise ValueError(f"dim mismatch on {l}")
    m = 1
    for l in fa:
        m *= dim[l]
    k = 1
    for l in common:
        k *= dim[l]
    n = 1
    for l in fb:
        n *= dim[l]
    a2 = permute(a, fa + common)[2].reshape(m, k)
    b2 = permute(b, common + fb)[2].reshape(k, n)
    c = (a2 @ b2).reshape(-1)
    return (tuple(fa + fb), tuple(dim[l] for l in fa + fb), c)


def to_device(leaves, device="cuda"):
    """(labels, dims, numpy array) leaves -> complex128 device tuples."""
    return [(tuple(l), tuple(d), torch.as_tensor(x).to(device=device, dtype=torch.complex128).reshape(-1))
            for l, d, x in leaves]


def run_schedule(leaves, steps, n_leaves, assignment):
    """steps: (lhs, rhs, result) SSA triples.  Returns the root tensor."""
    values = {}
    proj = {}
    for lhs_ref, rhs_ref, res in steps:
        ops = []
        for ref in (lhs_ref, rhs_ref):
            if ref < n_leaves:
                if ref not in proj:
                    proj[ref] = project(leaves[ref], assignment)
                ops.append(proj[ref])
            else:
                ops.append(values.pop(ref))
        values[res] = contract(ops[0], ops[1])
        del ops
    return values[steps[-1][2]]

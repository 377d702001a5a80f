"""Shared helpers of the GPU parity tests: upload synthetic inputs, unpack
device results into numpy for comparison with the oracle.  No method
arithmetic lives here."""
import numpy as np
import torch

import synth


def to_bf16_cuda(a):
    bits = synth.bf16_bits(a).view(np.int16)
    return torch.from_numpy(bits.copy()).view(torch.bfloat16).cuda()


def unpack_bits(words, cols):
    w = words.cpu().numpy().view(np.uint32).astype(np.uint64)
    bits = (w[..., None] >> np.arange(32, dtype=np.uint64)) & 1
    return bits.reshape(w.shape[0], -1)[:, :cols].astype(bool)


def rel_frob(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def code_mismatch(gpu_codes, oracle_codes):
    g = gpu_codes.astype(np.int64)
    o = oracle_codes.astype(np.int64)
    diff = np.abs(g - o)
    return int((diff > 0).sum()), int(diff.max(initial=0))


def item_pairs(items, wexp):
    """(item id, weight exponent) pairs sorted by item id: the kept set of an LSS
    mask, independent of the order a kernel stores its list in."""
    items = np.asarray(items, dtype=np.int64)
    wexp = np.asarray(wexp, dtype=np.int64)
    order = np.argsort(items, kind="stable")
    return np.stack([items[order], wexp[order]])


def same_item_set(gpu_items, gpu_wexp, ora):
    """The GPU's kept (item, weight) set equals the oracle mask `ora` exactly, and
    no item appears twice."""
    g = item_pairs(gpu_items, gpu_wexp)
    if g.shape[1] != ora["count"]:
        return False
    if g.shape[1] and np.any(np.diff(g[0]) == 0):
        return False
    return np.array_equal(g, item_pairs(ora["items"], ora["wexp"]))

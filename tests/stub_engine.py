"""TEST-ONLY CPU stand-in for the CUDA bucket engine, built on the oracle.

Lets the CPU suite exercise LagsSGD's host logic (fusion buckets, hook scheduling, release
order, all-gather plumbing over gloo, decode ordering) without a GPU.  It reproduces the CUDA
bucket's message layout byte for byte.  Never used by the product (which has no CPU path).
"""

import numpy as np
import torch

from oracle import lagsgd_oracle as orc


def _align(x, a=16):
    return (x + a - 1) // a * a


class OracleStubBucket:
    def __init__(self, dims, ks, world, device):
        self.dims = [int(d) for d in dims]
        self.ks = [int(k) for k in ks]
        self.nlayers = len(dims)
        self.offsets = np.concatenate([[0], np.cumsum(self.dims)[:-1]]).astype(np.int64)
        self.slots = np.concatenate([[0], np.cumsum(self.ks)[:-1]]).astype(np.int64)
        self.total_k = int(sum(self.ks))
        self.n_total = int(sum(self.dims))
        self.off_cnt = 0
        self.off_idx = _align(4 * self.nlayers)
        self.off_val = _align(self.off_idx + 4 * self.total_k)
        self.msg_bytes = _align(self.off_val + 4 * self.total_k)
        self.calls = 0

    def new_messages(self, count):
        return torch.zeros(count * self.msg_bytes, dtype=torch.uint8)

    def compress(self, g, r, alpha, msg, status, stream=None, exact=False, zero_grad=False):
        gn = g.detach().numpy()
        rn = r.detach().numpy()
        self.last_g = gn.copy()  # tests rebuild the gradient the optimizer consumed
        if not np.all(np.isfinite(gn)):
            status[0] |= 1
        raw = msg.numpy()
        cnt = raw[self.off_cnt:self.off_cnt + 4 * self.nlayers].view(np.int32)
        idx = raw[self.off_idx:self.off_idx + 4 * self.total_k].view(np.int32)
        val = raw[self.off_val:self.off_val + 4 * self.total_k].view(np.float32)
        for j, (d, k) in enumerate(zip(self.dims, self.ks)):
            o, s = self.offsets[j], self.slots[j]
            i, v = orc.compress_layer(gn[o:o + d], rn[o:o + d], float(alpha), k)
            cnt[j] = len(i)
            idx[s:s + len(i)] = i
            val[s:s + len(i)] = v
        if zero_grad:
            g.zero_()
        self.calls += 1

    def decode(self, msgs, P, v, momentum=None, mu=0.0, stream=None):
        total = np.zeros(self.n_total)
        raw = msgs.numpy()
        for p in range(P):
            m = raw[p * self.msg_bytes:(p + 1) * self.msg_bytes]
            cnt = m[self.off_cnt:self.off_cnt + 4 * self.nlayers].view(np.int32)
            idx = m[self.off_idx:self.off_idx + 4 * self.total_k].view(np.int32)
            val = m[self.off_val:self.off_val + 4 * self.total_k].view(np.float32)
            for j in range(self.nlayers):
                s, o = self.slots[j], self.offsets[j]
                total[o + idx[s:s + cnt[j]]] += val[s:s + cnt[j]]  # indices unique within a rank
        vn = v.detach().numpy()
        if mu:
            mn = momentum.detach().numpy()
            mn[:] = (mu * mn.astype(np.float64) + total / P).astype(np.float32)
            vn[:] = (vn.astype(np.float64) - mn.astype(np.float64)).astype(np.float32)
        else:
            vn[:] = (vn.astype(np.float64) - total / P).astype(np.float32)


    def reconstruct(self, msgs, P, r, acc, stream=None):
        raw = msgs.numpy()
        rn, an = r.detach().numpy(), acc.numpy()
        an[:P * self.n_total] = rn[:P * self.n_total]
        for p in range(P):
            m = raw[p * self.msg_bytes:(p + 1) * self.msg_bytes]
            cnt = m[self.off_cnt:self.off_cnt + 4 * self.nlayers].view(np.int32)
            idx = m[self.off_idx:self.off_idx + 4 * self.total_k].view(np.int32)
            val = m[self.off_val:self.off_val + 4 * self.total_k].view(np.float32)
            for j in range(self.nlayers):
                s, o = self.slots[j], self.offsets[j]
                an[p * self.n_total + o + idx[s:s + cnt[j]]] = val[s:s + cnt[j]]

    def delta(self, acc, r, P, out=None, stream=None):
        an = acc.numpy().reshape(P, self.n_total)
        res = []
        for j, (d, k) in enumerate(zip(self.dims, self.ks)):
            o = self.offsets[j]
            got = orc.topk_aggregation_ratio([an[p, o:o + d] for p in range(P)], k)
            res.append(float("nan") if got is None else got)
        t = torch.tensor(res, dtype=torch.float64)
        if out is not None:
            out.copy_(t)
            return out
        return t


def stub_factory(dims, ks, world, device):
    return OracleStubBucket(dims, ks, world, device)

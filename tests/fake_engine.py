"""CPU stand-in for multi_gpu.LibEngine, for the gloo tests of the multi-rank PROTOCOL only.

It implements the same step interface (vertex_max / claims / decide / check_commit /
exact_level / end_round / finish) with numpy and the oracle's priority stream, on torch CPU tensors
so that torch.distributed (gloo) can all-reduce them.  Test infrastructure: the product path is
LibEngine (CUDA kernels through the C-ABI); nothing in the package imports this file."""
import numpy as np
import torch

from oracle import pyoracle as po

MG_RUNNING, MG_DONE, MG_ROUND_LIMIT = 0, 1, 2


class FakeEngine:
    stream = None  # no CUDA stream

    def __init__(self, g: po.Graph, begin: int, count: int):
        self.g, self.b, self.k = g, begin, count
        self.n = g.n
        self.ids = np.arange(begin, begin + count, dtype=np.uint32)
        off = g.edge_offsets.astype(np.int64)
        self.rows = [g.edge_members[off[e]:off[e + 1]].astype(np.int64) for e in self.ids]
        self.base = g.base_weights[begin:begin + count]
        self.nw, self.nc = (self.n + 31) // 32, (self.n + 7) // 8
        self.vkey = torch.zeros(self.n, dtype=torch.int64)
        self.exch = torch.zeros(self.nw + self.nc + 8, dtype=torch.int32)
        self.exact = None
        self.orc = po.Oracle("port")

    def keys(self):
        return self.vkey

    def claims_and_stats(self):
        return self.exch[self.nw:]

    def dead_new(self):
        return self.exch[:self.nw]

    def sync(self):
        pass

    def weight_info(self, lo):
        if self.k == 0:
            return 1.0, 1.0, 0, 0
        w = self.base + lo
        return float(self.base.min()), float(self.base.max()), int(np.any(w != np.floor(w))), self.k

    def begin(self, stream, cfg, bmin, bmax, nonint, m_global):
        self.s = po.Stream(stream.seed, {"xorshift": 0, "park_miller": 1, "splitmix": 2}[stream.kind],
                           {"perturb_base": 0, "replace_uniform": 1}[stream.mode], stream.noise_low, stream.noise_high)
        self.max_rounds = cfg.max_rounds or self.orc.default_max_rounds(m_global)
        self.active = np.ones(self.k, dtype=bool)
        self.dead = np.zeros(self.n, dtype=bool)
        self.round = 1
        self.mround = np.zeros(self.k, dtype=np.uint16)
        self.matched_r, self.dropped_r = [], []
        self.vkey.zero_()
        self.exch.zero_()
        self.limit = False
        self.rounds_done = 0

    def _keys_now(self):
        idx = np.nonzero(self.active)[0]
        w, t = self.orc.eval_stream(self.s, self.ids[idx], np.full(idx.size, self.round, dtype=np.uint32), self.base[idx])
        return idx, w.view(np.int64).copy(), t

    def vertex_max(self):
        dropped = 0
        for i in np.nonzero(self.active)[0]:
            if self.dead[self.rows[i]].any():
                self.active[i] = False
                dropped += 1
        if self.round > 1:
            self.dropped_r.append(dropped)
        self.idx, self.kw, self.kt = self._keys_now()
        vk = np.zeros(self.n, dtype=np.int64)
        for j, i in enumerate(self.idx):
            np.maximum.at(vk, self.rows[i], self.kw[j])
        self.vkey.copy_(torch.from_numpy(vk))  # keys of this round only (no tags in the stand-in)

    def claims(self):
        vk = self.vkey.numpy()
        claims = np.zeros(self.n, dtype=np.int64)
        for j, i in enumerate(self.idx):
            rows = self.rows[i]
            np.add.at(claims, rows[vk[rows] == self.kw[j]], 1)
        packed = np.zeros(self.nc, dtype=np.int64)
        v = np.nonzero(claims)[0]
        np.add.at(packed, v >> 3, np.minimum(claims[v], 15) << ((v & 7) * 4))
        self.exch[self.nw:self.nw + self.nc] = torch.from_numpy(packed.astype(np.uint32).view(np.int32))
        self.exch[self.nw + self.nc] = int(self.idx.size)
        self.exch[self.nw + self.nc + 1] = 0

    def decide(self):
        words = self.exch[self.nw:self.nw + self.nc].numpy().view(np.uint32)
        tie = bool(np.any(words & 0xEEEEEEEE))
        return int(self.exch[self.nw + self.nc].item()), tie

    def _commit(self, winners):
        bits = np.zeros(self.nw, dtype=np.uint32)
        for i in winners:
            self.active[i] = False
            self.mround[i] = self.round
            rows = self.rows[i]
            np.bitwise_or.at(bits, rows >> 5, (1 << (rows & 31)).astype(np.uint32))
        self.exch[:self.nw] = torch.from_numpy(bits.view(np.int32))
        self._matched_now = len(winners)

    def check_commit(self):
        if self.round > self.max_rounds:
            self._matched_now = 0
            return
        vk = self.vkey.numpy()
        self._commit([i for j, i in enumerate(self.idx) if np.all(vk[self.rows[i]] == self.kw[j])])

    def exact_arrays(self):
        if self.exact is None:
            self.exact = (torch.zeros(self.n, dtype=torch.int64), torch.zeros(self.n, dtype=torch.int64),
                          torch.zeros(self.n, dtype=torch.int32))
        return self.exact

    def exact_level(self, level):
        va, vb, vc = (a.numpy() for a in self.exact_arrays())
        vbu, vcu = vb.view(np.uint64), vc.view(np.uint32)
        if self.round > self.max_rounds:
            self._matched_now = 0
            return
        winners = []
        for j, i in enumerate(self.idx):
            rows, A, B, Cc = self.rows[i], self.kw[j], self.kt[j], np.uint32(self.ids[i] + 1)
            if level == 1:
                np.maximum.at(va, rows, A)
            elif level == 2:
                np.maximum.at(vbu, rows[va[rows] == A], B)
            elif level == 3:
                np.maximum.at(vcu, rows[(va[rows] == A) & (vbu[rows] == B)], Cc)
            elif np.all((va[rows] == A) & (vbu[rows] == B) & (vcu[rows] == Cc)):
                winners.append(i)
        if level == 4:
            self._commit(winners)

    def end_round(self, global_active):
        bits = self.exch[:self.nw].numpy().view(np.uint32)
        v = np.nonzero(np.unpackbits(bits.view(np.uint8), bitorder="little")[:self.n])[0]
        self.dead[v] = True
        self.exch.zero_()
        if global_active == 0:
            self.rounds_done = self.round - 1
            return MG_DONE
        if self.round > self.max_rounds:
            self.rounds_done = self.round - 1
            self.limit = True
            return MG_ROUND_LIMIT
        self.matched_r.append(self._matched_now)
        self.round += 1
        return MG_RUNNING

    def finish(self, weight_before):
        sel = np.nonzero(self.mround)[0]
        tw = weight_before
        for i in sel:
            tw += self.base[i]
        r = self.rounds_done
        matched = np.array(self.matched_r[:r], dtype=np.int64)
        dropped = np.array(self.dropped_r[:r], dtype=np.int64)
        return dict(matched=self.ids[sel], round_of=self.mround[sel], per_round_matched=matched,
                    per_round_deactivated=dropped, rounds=r, total_weight=float(tw), launches=0,
                    tie_redos=0, limit=self.limit)

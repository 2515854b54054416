"""numpy restatement of the edge-partitioned round protocol of csrc/hlm_shard.inc, for the gloo tests.

Same steps, same arrays crossing ranks, same decisions -- local argmax under the full comparator, keys of
the LIVE vertices in slot order, all-reduce(max), owner count against the number of vertices with a
maximum, the three tie levels, edge-side agreement, covered bitmap + statistics all-reduce(sum), kill,
alive count, live-set update -- with the collectives handed in as callbacks (torch.distributed/gloo in
tests/test_multi_protocol_gloo.py).  Test infrastructure: the product path is the CUDA library; nothing in
the package imports this file."""
import numpy as np

from oracle import pyoracle as po

NONE = -1


class ShardModel:
    def __init__(self, g: po.Graph, begin: int, count: int, stream: po.Stream, allreduce_max, allreduce_sum,
                 max_rounds: int = 0, exact_always: bool = False):
        self.g, self.b, self.k, self.s = g, begin, count, stream
        self.n = g.n
        self.amax, self.asum = allreduce_max, allreduce_sum
        self.exact_always = exact_always
        self.orc = po.Oracle("port")
        off = g.edge_offsets.astype(np.int64)
        self.rows = [g.edge_members[off[e]:off[e + 1]].astype(np.int64) for e in range(begin, begin + count)]
        self.base = g.base_weights[begin:begin + count]
        m_global = int(self.asum(np.array([count], dtype=np.int64))[0])
        self.m_global = m_global
        self.max_rounds = max_rounds or self.orc.default_max_rounds(m_global)

    def _local_argmax(self, alive, live, r):
        """per vertex: (weight bits, tie hash, global id) of the best alive local edge, NONE if none"""
        idx = np.nonzero(alive)[0]
        gids = (idx + self.b).astype(np.uint32)
        w, t = self.orc.eval_stream(self.s, gids, np.full(idx.size, r, dtype=np.uint32), self.base[idx])
        wb = w.view(np.int64)  # positive doubles: the bit pattern orders like the value
        best = {}
        for j, i in enumerate(idx):
            key = (int(wb[j]), int(t[j]), int(gids[j]))
            for v in self.rows[i]:
                if live[v] and (v not in best or key > best[v][0]):
                    best[v] = (key, i)
        return best

    def run(self):
        n = self.n
        alive = np.ones(self.k, dtype=bool)
        live = np.ones(n, dtype=bool)
        mround = np.zeros(self.k, dtype=np.uint16)
        active = self.m_global
        rounds, tie_redos, limit = 0, 0, False
        prm, prd, live_r, bytes_r = [], [], [], []
        while active > 0:
            rounds += 1
            if rounds > self.max_rounds:
                limit = True
                rounds -= 1
                break
            r = rounds
            slots = np.cumsum(live) - 1  # slot of a live vertex = its rank among the live ones
            L = int(live.sum())
            best = self._local_argmax(alive, live, r)
            lkey = np.zeros(L, dtype=np.int64)
            top = np.full(n, NONE, dtype=np.int64)
            for v, (key, i) in best.items():
                lkey[slots[v]] = key[0]
                top[v] = i
            gkey = self.amax(lkey.copy())
            expected = int(np.count_nonzero(gkey))
            lv = np.nonzero(live)[0]
            own = (lkey != 0) & (lkey == gkey)
            claims = int(self.asum(np.array([np.count_nonzero(own)], dtype=np.int64))[0])
            moved = L * 8
            tie = claims != expected
            if tie or self.exact_always:
                tie_redos += int(tie and not self.exact_always)
                # level 2: tie hash among the weight owners (uint64 order through int64: flip the sign bit)
                h = np.zeros(L, dtype=np.int64)
                for v in lv[own]:
                    h[slots[v]] = np.int64(np.uint64(best[v][0][1]) ^ np.uint64(1 << 63))
                h[~own] = np.iinfo(np.int64).min
                g2 = self.amax(h.copy())
                own2 = own & (h == g2)
                # level 3: global id + 1 among the (weight, hash) owners
                ident = np.zeros(L, dtype=np.int64)
                for v in lv[own2]:
                    ident[slots[v]] = best[v][0][2] + 1
                g3 = self.amax(ident.copy())
                own = own2 & (ident == g3)
                claims = int(self.asum(np.array([np.count_nonzero(own)], dtype=np.int64))[0])
                assert claims == expected, "after the exact levels every maximum has one owner"
                moved += 2 * L * 8
            top[lv[~own]] = NONE
            # agreement from the edge side; covered bitmap + matched count cross ranks
            covered = np.zeros((n + 31) // 32 + 1, dtype=np.int64)
            matched_now = []
            for i in np.nonzero(alive)[0]:
                if np.all(top[self.rows[i]] == i):
                    matched_now.append(i)
                    rr = self.rows[i]
                    np.bitwise_or.at(covered, rr >> 5, np.int64(1) << (rr & 31))
            covered[-1] = len(matched_now)
            covered = self.asum(covered)
            matched_total = int(covered[-1])
            moved += ((n + 31) // 32 + 8) * 4
            cov = ((covered[:-1][np.arange(n) >> 5] >> (np.arange(n) & 31)) & 1).astype(bool)
            for i in matched_now:
                alive[i] = False
                mround[i] = r
            for i in np.nonzero(alive)[0]:
                if cov[self.rows[i]].any():
                    alive[i] = False
            alive_total = int(self.asum(np.array([np.count_nonzero(alive)], dtype=np.int64))[0])
            moved += 16
            has_max = np.zeros(n, dtype=bool)
            has_max[lv] = gkey != 0
            prm.append(matched_total)
            prd.append(active - alive_total - matched_total)
            live_r.append(L)
            bytes_r.append(moved)
            active = alive_total
            live = live & has_max & ~cov
        sel = np.nonzero(mround)[0]
        return dict(matched=(sel + self.b).astype(np.uint32), round_of=mround[sel], weights=self.base[sel], per_round_matched=prm,
                    per_round_deactivated=prd, rounds=rounds, live=live_r, bytes=bytes_r, tie_redos=tie_redos, limit=limit)

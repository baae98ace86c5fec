"""TEST INFRASTRUCTURE: a CPU store with the ops.ChunkStore lookup_insert
contract, restating the reference's first-writer-wins dict
(registry.py:126-140) for the multi-process (gloo) tests of shard.py."""

import torch


class DictStore:
    def __init__(self, max_entries: int = 1 << 16):
        self.map: dict[int, int] = {}
        self.e_p_src = torch.zeros(max_entries, dtype=torch.int64)
        self.e_row = torch.zeros(max_entries, dtype=torch.int64)
        self.rows = 0

    def lookup_insert(self, q_fp, q_order, q_p, q_len, q_probe=None):
        n = q_fp.numel()
        assert bool((q_order[1:] > q_order[:-1]).all()) if n > 1 else True, "q_order must ascend"
        hit = torch.full((n,), -1, dtype=torch.int32)
        entry = torch.full((n,), -1, dtype=torch.int64)
        p_src = torch.zeros(n, dtype=torch.int64)
        row = torch.full((n,), -1, dtype=torch.int64)
        for i in range(n):
            if q_probe is not None and not q_probe[i]:
                continue
            f = int(q_fp[i])
            e = self.map.get(f)
            if e is None:
                e = len(self.map)
                self.map[f] = e
                self.e_p_src[e] = int(q_p[i])
                self.e_row[e] = self.rows
                self.rows += int(q_len[i])
                hit[i] = 0
            else:
                hit[i] = 1
            entry[i] = e
            p_src[i] = self.e_p_src[e]
            row[i] = self.e_row[e]
        return hit, entry, p_src, row

"""Dependency depth of the waiting heavy pass (tooling): the longest chain of
heavy rows (degree >= T) each adjacent to the next with ascending ids, i.e.
the critical path of K1HW in row commits.  Level-synchronous relaxation on
the GPU with torch.
    python tools/chain_depth.py rmat24 [T ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1505_04086_b200 import graphs
    cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
    Ts = [int(x) for x in sys.argv[2:]] or [64, 1024]
    off, cols = graphs.make_config(cfg, "cuda")
    n = off.numel() - 1
    deg = (off[1:] - off[:-1])
    rows = torch.repeat_interleave(torch.arange(n, device="cuda", dtype=torch.int32), deg)
    for T in Ts:
        heavy = deg >= T
        keep = heavy[rows.long()] & heavy[cols.long()] & (cols < rows)
        r, c = rows[keep].long(), cols[keep].long()
        depth = heavy.to(torch.int32)
        t0 = time.time()
        it = 0
        while True:
            it += 1
            new = depth.clone()
            new.scatter_reduce_(0, r, depth[c] + 1, "amax")
            if torch.equal(new, depth):
                break
            depth = new
        print(f"{cfg} T={T}: heavy rows {int(heavy.sum())}, lower heavy-heavy entries {r.numel()}, "
              f"longest chain {int(depth.max())} rows ({it} sweeps, {time.time() - t0:.1f} s)", flush=True)
        # how the chain splits: members that are split rows (degree >= 1024)
        if T < 1024:
            v = int(depth.argmax())
            hubs = 0
            d = int(depth[v])
            cur = v
            while d > 1:
                lo, hi = int(off[cur]), int(off[cur + 1])
                nb = cols[lo:hi].long()
                nb = nb[(nb < cur) & heavy[nb]]
                nxt = nb[depth[nb] == d - 1][0]
                hubs += int(deg[cur] >= 1024)
                cur, d = int(nxt), d - 1
            print(f"  one longest chain: {hubs} of its {int(depth.max())} rows have degree >= 1024", flush=True)


if __name__ == "__main__":
    main()

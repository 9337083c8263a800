"""Summarise PP_PROFILE_DUMP output (one line per timed launch: band cat us GFLOP) per step position."""
import collections
import sys

L = [l.split() for l in open(sys.argv[1])]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
n = len(L) // steps
pos = collections.defaultdict(list)
for i, l in enumerate(L[: n * steps]):
    pos[i % n].append(float(l[2]))
cats = {0: "conv", 1: "gemm", 2: "gn", 3: "other"}
tot = 0
for k in range(n):
    v = sorted(pos[k])[len(pos[k]) // 2]
    tot += v
    l = L[n * (steps // 2) + k]
    fl = float(l[3])
    tf = fl / (v * 1e-6) / 1e3 if fl > 0 else 0
    print(f"{k:3d} {cats.get(int(l[1]), l[1]):5s} {v:8.2f} us {fl:8.2f} GF {tf:6.0f} TF/s")
print(f"launches/step {n}  sum of medians {tot:.1f} us")

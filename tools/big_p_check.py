"""Large-p check: python tools/big_p_check.py 70000 24 -- 2.45e9 pairs (slots past 2^31),
19.6 GB of output, sampled pairs against the oracle."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle
from paper_2307_04904_b200 import api, generators as gen
p, L = int(sys.argv[1]), int(sys.argv[2])
rng = gen.SplitMix64(11)
samples = rng.gaussian(p * L)
offsets = np.arange(p + 1, dtype=np.int64) * L
t0 = time.time()
m = api.build_matrix_packed(samples, offsets, api.WarpWindow(None), False)
t1 = time.time()
D = m.condensed()
total = p * (p - 1) // 2
print("p", p, "pairs", total, "build s", round(t1 - t0, 2), "bytes", D.nbytes, flush=True)
r = np.random.default_rng(0)
idx = r.integers(0, total, size=200)
idx = np.concatenate([idx, [0, total - 1, 2**31 - 1 if total > 2**31 else total // 2, 2**31 if total > 2**31 + 1 else total // 3]])
def decode(s):
    lo, hi = 0, p - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if mid * p - mid * (mid + 1) // 2 <= s: lo = mid
        else: hi = mid - 1
    i = lo
    return i, i + 1 + (s - (i * p - i * (i + 1) // 2))
bad = 0
for s in idx:
    i, j = decode(int(s))
    want = oracle.dtw(samples[i*L:(i+1)*L], samples[j*L:(j+1)*L], -1)
    bad += int(D[int(s)] != want)
print("sampled", len(idx), "mismatches", bad)

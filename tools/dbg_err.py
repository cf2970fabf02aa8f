import sys; sys.path.insert(0, '/root/repo')
import numpy as np, paper_1209_5198_b200 as f2
from oracle import pyoracle as po
ctx = f2.Context(0)
for (n, m) in [(64, 64), (200, 130), (1, 1)]:
    a = po.random_dense(n, m, 0.5, 3)
    try:
        got = f2.decompose_block(f2.BitMatrix(n, m, a), ctx=ctx)
        print(n, m, "ok rank", got.rank)
    except Exception as e:
        print(n, m, "ERR", e)

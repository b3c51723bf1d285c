"""Host packing rate of one c3 batch (InputLayout.pack -> dlrm_pack_batch) by thread count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from concurrent.futures import ThreadPoolExecutor
from paper_1906_00091_b200.pipeline import InputLayout
from paper_1906_00091_b200.rng import RandomBatchSource
src = RandomBatchSource([10**6]*8, 512, 2048, 100, False, seed=1)
hb = src.next_batch()
caps = [len(i) for i in hb.indices]
L = InputLayout(2048, 8, 512, caps, False)
import torch
blk = L.new_host_block() if torch.cuda.is_available() else torch.zeros(L.nbytes, dtype=torch.uint8)
for th in (1, 2, 4, 6, 8, 12, 16):
    pool = ThreadPoolExecutor(th)
    for _ in range(3): L.pack(blk, hb.dense, hb.offsets, hb.indices, hb.labels, None, pool)
    t=time.perf_counter()
    for _ in range(30): L.pack(blk, hb.dense, hb.offsets, hb.indices, hb.labels, None, pool)
    print(th, round((time.perf_counter()-t)/30*1e3, 3), 'ms')

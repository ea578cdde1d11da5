import sys, collections
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
torch.cuda.set_device(0)
import paper_1806_08020_b200 as ppa
ppa.set_stream(torch.cuda.current_stream())
from test_gpu_fuzz_layouts import _case
cnt = collections.Counter()
for seed in range(48):
    n, rows, cols, vals = _case(seed)
    P = ppa.CsrMatrix.from_triplets(n, rows, cols, vals)
    for cap in ("auto", "sell32_packed", "dia_coded"):
        L = ppa.make_csr_operator(P, cap).layout()
        cnt[(cap, L["layout"], L["sigma"] > 1, L["dict_size"] > 0)] += 1
for k, v in sorted(cnt.items()): print(k, v)

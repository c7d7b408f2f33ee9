import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_23043_b200 as T
from torch.profiler import profile, ProfilerActivity
f = T.Former(seed=1, scale=1.0, max_len=1024)
B, Tn = 4096, 784
rs = np.random.default_rng(0)
tok = rs.integers(0, 2, (B, Tn)).astype(np.uint8); betas = rs.uniform(0.2, 3, B)
f.log_prob(tok, betas, 48); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    f.log_prob(tok, betas, 48); torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=15))

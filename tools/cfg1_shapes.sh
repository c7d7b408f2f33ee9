# Config 1 launch shapes: K1 threads per CTA (TAPT_K1_THREADS) at the workload's 296 seeds, and 592 seeds.
for th in 128 256 512; do
  for I in 296 592; do
    echo "threads $th seeds $I: $(TAPT_K1_THREADS=$th python -c "
import sys, torch; sys.path.insert(0, '.')
import paper_2509_23043_b200 as T
from paper_2509_23043_b200 import workloads as WL
s = torch.cuda.Stream(); w = WL.build(T, 1, s.cuda_stream, instances=$I); w['step']()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record(s); w['step'](); b.record(s); torch.cuda.synchronize()
print(round(w['updates_per_step'] / (a.elapsed_time(b) * 1e-3) / 1e9, 1), 'G/s')")"
  done
done

#!/bin/bash
# projection experiments: per-launch cost vs batch size, CTA-0 timeline (trace build), H2D bandwidth
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for b in 512 2048 8192; do python tools/profile_ingest.py --config medium --batches $((16384/b)) --batch $b --reps 3 --synthetic-counts 2>&1 | tail -2; done
python - <<'PY'
import torch,time
x=torch.empty(512<<20,dtype=torch.uint8).pin_memory(); y=torch.empty_like(x,device='cuda')
for _ in range(3): y.copy_(x,non_blocking=True)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); [y.copy_(x,non_blocking=True) for _ in range(5)]; e1.record(); torch.cuda.synchronize()
print("H2D pinned GB/s", 5*x.numel()/e0.elapsed_time(e1)/1e6)
PY
WDD_NVCC_EXTRA=-DWDD_TRACE python -m paper_2212_01309_b200.build --force > /dev/null 2>&1
python tools/trace_proj.py medium 512 > gpurun_out/trace_512.txt 2>&1
python tools/trace_proj.py medium 8192 > gpurun_out/trace_8192.txt 2>&1
tail -12 gpurun_out/trace_512.txt; tail -12 gpurun_out/trace_8192.txt
python -m paper_2212_01309_b200.build --force > /dev/null 2>&1

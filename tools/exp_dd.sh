#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
WDD_FLUSH=gemm timeout 600 ncu --set full --clock-control none -k regex:"colgemm" -c 1 -o gpurun_out/r01dd_colgemm -f python tools/bench_live.py --config live --reps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r01dd_colgemm.ncu-rep
ncu -i gpurun_out/r01dd_colgemm.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; u=rows[1]
for r in rows[2:]:
  for i,k in enumerate(h):
    if any(t in k for t in ['l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sector_hit_rate','lts__t_sectors_srcunit_tex_op_read.sum','smsp__sass_inst_executed_op_shared','l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','l1tex__t_requests_pipe_lsu_mem_global_op_st.sum']) and not k.endswith('per_second') and 'pct' not in k: print(k, r[i], u[i])
"

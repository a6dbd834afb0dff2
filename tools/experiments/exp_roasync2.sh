# pipelined readouts: acquisitions per graph (Medium, Box), eager (no graph) Medium
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
run() { c=$1; shift; timeout 400 python bench.py --config $c --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/ra.json 2>gpurun_out/ra.err
  python -c "
import json;d=json.load(open('gpurun_out/ra.json'))
print('$c $*', '%.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'step %.3f'%d['step_roofline']['frac'])" || tail -3 gpurun_out/ra.err; }
for A in 1 4 8 16; do for v in 0 1; do run medium --steps 320 --acq-per-graph $A --readout-async $v; done; done
run medium --steps 320 --no-graph --readout-async 0
run medium --steps 320 --no-graph --readout-async 1
for A in 1 2; do for v in 0 1; do run box --steps 20 --acq-per-graph $A --readout-async $v; done; done
for A in 1 4 8; do run large --steps 48 --acq-per-graph $A --readout-async 1; done

#!/bin/bash
# Round-end evidence on one GPU (dev tool): smoke, every bench config, the
# reference arm, and the ncu launch list of the default bench command.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
for w in cfg2 cfg1 cfg3 cfg4 cfg5; do
  python bench.py --workload $w > gpurun_out/bench_$w.jsonl 2> gpurun_out/bench_$w.err
done
python bench.py --impl reference > gpurun_out/bench_reference_cfg2.jsonl 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-verify \
  > gpurun_out/ncu_launches.log 2>&1
tail -1 gpurun_out/smoke.log

#!/bin/bash
# ncu captures at BENCH sizes (one report per BASELINE config), each after a
# plain run of the same command; then per-config summaries via
# tools/ncu_summary.py (run here, not on the box).
set -u
mkdir -p gpurun_out
P=tools/prof_one.py
declare -A L=(
 [cfg2]="exp_d_u10@2@28,exp_d_u35@2@28,log_d_u10@2@28,log_d_u35@2@28,pow_d_u10@2@28,pow_d_u35@2@28,exp_f_u10@2@28,exp_f_u35@2@28,log_f_u10@2@28,log_f_u35@2@28,pow_f_u10@2@28,pow_f_u35@2@28"
 [cfg1]="sin_d_u10@1@24,cos_d_u10@1@24"
 [cfg3]="sin_d_u10_ph@3@28,cos_d_u10_ph@3@28,tan_d_u10_ph@3@28,sin_f_u10_ph@3@28,cos_f_u10_ph@3@28,tan_f_u10_ph@3@28"
 [cfg4]="fmod_d@4@26,fmod_f@4@26"
 [cfg5]="sin_d_u10@5@31,cos_d_u10@5@31,tan_d_u10@5@31,atan_d_u10@5@31,exp_d_u10@5@31,log_d_u10@5@31,pow_d_u10@5@31,fmod_d@5@31"
)
for w in ${CFGS:-cfg2 cfg1 cfg3 cfg4 cfg5}; do
  n=$(echo "${L[$w]}" | tr ',' '\n' | wc -l)
  python $P "${L[$w]}" 2 24 0 > gpurun_out/cap_${w}_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_trig|k_queue" -c $n \
      -o gpurun_out/r02_full_${w} python $P "${L[$w]}" 2 24 0 > gpurun_out/cap_${w}_ncu.log 2>&1
  echo "$w rc=$?"
done
# summarise on the box (reports are too large to bring back): per-config
# markdown + json, per-line attribution of the heaviest kernels; then drop
# the reports
for w in ${CFGS:-cfg2 cfg1 cfg3 cfg4 cfg5}; do
  case $w in cfg2|cfg3) n=$((1<<28));; cfg1) n=$((1<<24));; cfg4) n=$((1<<26));; cfg5) n=$((1<<31));; esac
  [ -f gpurun_out/r02_full_${w}.ncu-rep ] || continue
  python tools/ncu_summary.py gpurun_out/r02_full_${w}.ncu-rep $n gpurun_out/r02_full_${w} @$w > /dev/null 2>&1
  for k in ${LINES:-}; do
    python tools/ncu_lines.py gpurun_out/r02_full_${w}.ncu-rep "$k" $n >> gpurun_out/r02_lines_${w}.txt 2>&1
  done
  [ -n "${KEEP_REP:-}" ] || rm -f gpurun_out/r02_full_${w}.ncu-rep
done

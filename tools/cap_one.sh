#!/bin/bash
# quick ncu capture of a few entry points: bash tools/cap_one.sh LIST KERNEL_REGEX... (LIST as for prof_one.py, sizes 2^28)
set -u
LIST=$1; shift
mkdir -p gpurun_out
n=$(echo "$LIST" | tr ',' '\n' | wc -l)
python tools/prof_one.py "$LIST" 2 24 0 > gpurun_out/cap1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_trig|k_queue" -c $n -o gpurun_out/cap1 python tools/prof_one.py "$LIST" 2 24 0 > gpurun_out/cap1_ncu.log 2>&1
echo rc=$?
python tools/ncu_brief.py gpurun_out/cap1.ncu-rep $((1<<28)) > gpurun_out/cap1_brief.txt 2>&1
: > gpurun_out/cap1_lines.txt
for k in "$@"; do python tools/ncu_lines.py gpurun_out/cap1.ncu-rep "$k" $((1<<28)) >> gpurun_out/cap1_lines.txt 2>&1; done
rm -f gpurun_out/cap1.ncu-rep
cat gpurun_out/cap1_brief.txt

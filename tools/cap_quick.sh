set -u
mkdir -p gpurun_out
P=tools/prof_one.py
LIST="sin_d_u10@5@28,tan_d_u10@5@28,atan_d_u10@5@28,pow_d_u10@5@28,fmod_d@5@28,sin_f_u10@3@28,tan_f_u10@3@28,sin_d_u10_ph@3@28,tan_d_u10_ph@3@28,fmod_f@4@26,pow_d_u10@2@28,log_f_u10@2@28,pow_f_u10@2@28,sin_d_u10@1@24"
n=$(echo "$LIST" | tr ',' '\n' | wc -l)
python $P "$LIST" 2 24 0 > gpurun_out/capq_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_stream|k_trig|k_queue" -c $n -o gpurun_out/capq python $P "$LIST" 2 24 0 > gpurun_out/capq_ncu.log 2>&1
echo rc=$?
python tools/ncu_brief.py gpurun_out/capq.ncu-rep $((1<<28)) > gpurun_out/capq_brief.txt 2>&1
for k in "k_trig<vem::OpSinD," "k_trig<vem::OpTanD," "OpAtanD," "OpPowD," "FmodQ" "OpSinF" "OpTanF" "OpSinDPh" "OpFmodFFlat" "OpLogF," "OpPowF,"; do
  python tools/ncu_lines.py gpurun_out/capq.ncu-rep "$k" $((1<<28)) >> gpurun_out/capq_lines.txt 2>&1
done
rm -f gpurun_out/capq.ncu-rep

python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt; cat gpurun_out/launches.txt
ncu --nvtx --nvtx-include "step/" --set full --clock-control none --import-source on -k regex:k_accum_aff -c 1 -o gpurun_out/prof_accum -f python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; echo "ncu full rc $?"
ncu --nvtx --nvtx-include "step/" --set full --clock-control none --import-source on -k regex:k_digits_v -c 2 -o gpurun_out/prof_digits -f python tools/profile_step.py > gpurun_out/ncu3.log 2>&1; echo "ncu full2 rc $?"

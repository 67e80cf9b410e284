# config-3 bench line + the step's launch list
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
ncu --nvtx --nvtx-include "step/" --cache-control none --clock-control none -k regex:k_accum_aff --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/accum_traffic.csv python tools/profile_step.py > gpurun_out/ncu2.log 2>&1
ncu --nvtx --nvtx-include "step/" --set full --clock-control none --import-source on -k regex:k_accum_aff -c 1 -o gpurun_out/prof_accum -f python tools/profile_step.py > gpurun_out/ncu3.log 2>&1; echo "ncu full rc $?"

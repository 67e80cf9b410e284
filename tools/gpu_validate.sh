# round-end validation on one GPU: the whole -m gpu suite, smoke(), the default bench line and
# a K = 20 bench line, the lone-step launch list (all under gpurun_out/)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc $?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err; echo "bench k20 rc $?"
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt; head -8 gpurun_out/launches.txt

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
for v in "X=1" "TC_MSM_GENERIC_DIGITS=1" "TC_MSM_T1=16"; do
env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-monomial --no-cpu --no-forward > gpurun_out/ab.json 2>gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
done
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv | head -12

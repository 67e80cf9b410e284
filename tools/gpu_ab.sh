timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config3 or float_exponent or host_inputs" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for v in "TC_MSM_NC=1" "TC_MSM_NC=4" "TC_MSM_NC=8" "TC_MSM_NC=16" "TC_MSM_NC=32"; do
env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-monomial --no-cpu --no-forward > gpurun_out/ab.json 2>gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
done

timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "quantize or config3 or host_inputs or config1" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_gpu.log
for v in "X=1" "TC_MSM_SEG_LG=2" "TC_MSM_SEG_LG=4" "TC_MSM_SEG_LG=5"; do
env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-monomial --no-cpu --no-forward > gpurun_out/ab.json 2>gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
done

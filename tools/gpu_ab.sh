timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
for v in "X=1" "TC_MSM_FP_MIN_N=1000000000"; do
env $v TC_MSM_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-monomial --no-cpu --no-forward > gpurun_out/ab.json 2>gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['roofline']['work'].split(' x')[0], d['root'][:16])"
grep "L=32" gpurun_out/ab.err | head -2
done

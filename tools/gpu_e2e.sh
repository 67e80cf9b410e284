timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_inputs or commit_stream" > gpurun_out/pytest_host.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_host.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-monomial --no-cpu --no-forward > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo "bench rc $?"
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['ms_per_step'], json.dumps(d['e2e']))"
tail -3 gpurun_out/bench_e2e.err

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_gpu.log
for nl in 4 32; do TC_PROFILE_TIME=1 TC_PROFILE_LAYERS=$nl python tools/profile_step.py 2>&1 | tail -1; done

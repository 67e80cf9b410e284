timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_gpu.log
python tools/determinism.py 2>&1 | tail -1
for v in "X=1" "TC_MSM_NO_BLK_DIGITS=1"; do
for nl in 4 32; do env $v TC_PROFILE_TIME=1 TC_PROFILE_LAYERS=$nl python tools/profile_step.py 2>&1 | tail -1 | sed "s/^/$v /"; done
done
TC_PROFILE_CONFIG=5 TC_PROFILE_LAYERS=6 TC_PROFILE_TIME=1 python tools/profile_step.py 2>&1 | tail -1
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv | head -6

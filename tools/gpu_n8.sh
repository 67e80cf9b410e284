# per-rank work of an 8-GPU config-3 step (4 layers) and of a 4-GPU step (8 layers)
for nl in 4 8; do
TC_PROFILE_LAYERS=$nl python tools/profile_step.py > gpurun_out/plain_$nl.log 2>&1 && \
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$nl.csv env TC_PROFILE_LAYERS=$nl python tools/profile_step.py > gpurun_out/ncu_$nl.log 2>&1
echo "== layers $nl"; python tools/launch_summary.py gpurun_out/launches_$nl.csv | tail -12
done

# step launch list + full captures of the mode-1 counting-sort passes and the Newton interpolation
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches.txt
ncu --nvtx --nvtx-include "step/" --set full --clock-control none --import-source on -k regex:k_fpb_pass -c 2 -o gpurun_out/prof_fpb -f python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; echo "ncu fpb rc $?"
ncu --set full --clock-control none --import-source on -k regex:k_interp_newton -c 2 -o gpurun_out/prof_interp -f python tools/profile_mono.py > gpurun_out/ncu3.log 2>&1; echo "ncu interp rc $?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log

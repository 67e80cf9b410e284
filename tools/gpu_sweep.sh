for rep in 1 2; do for v in "TC_MSM_T=16" "TC_MSM_T=24" "TC_MSM_T=32" "TC_MSM_T=32 TC_MSM_T1=16" "TC_MSM_T=16 TC_MSM_T1=16"; do
env $v TC_PROFILE_TIME=1 python tools/profile_step.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done

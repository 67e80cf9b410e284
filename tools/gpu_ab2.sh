for lib in paper_2602_12630_b200/libtcb200.so abvar/lib_st1.so abvar/lib_st2.so; do
TC_LIB=$PWD/$lib python tools/profile_step.py > gpurun_out/plain.log 2>&1 && TC_LIB=$PWD/$lib ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_digits_fp --log-file gpurun_out/l.csv python tools/profile_step.py > /dev/null 2>&1
echo $lib; grep -E "k_digits_fp" gpurun_out/l.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160
done

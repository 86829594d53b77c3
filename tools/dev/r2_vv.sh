for m in 0 1 2; do
  GM_DEBUG_CONFIG=ls_mode=$m timeout -s KILL 200 python tools/dev/dev_fc_ops.py 2>&1 | head -1 > gpurun_out/r2vv_m$m.log
  GM_DEBUG_CONFIG=ls_mode=$m timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:line_sums -c 6 --csv python tools/dev/dev_fc_ops.py > gpurun_out/r2vv_ncu_m$m.csv 2>&1
  echo "mode $m"; cat gpurun_out/r2vv_m$m.log; grep -E "gpu__time_duration" gpurun_out/r2vv_ncu_m$m.csv | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
done

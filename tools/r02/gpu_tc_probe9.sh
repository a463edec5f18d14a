out=gpurun_out/r02_tc_probe9.log
: > $out
for v in "GFT_TC_LOAD_PACE_NS=2300" "GFT_TC_LOAD_PACE_NS=2500" "" "GFT_TC_LOAD_PACE_NS=2600" "GFT_TC_LOAD_PACE_NS=2800" "GFT_TC_LOAD_PACE_NS=2450"; do
  env $v timeout 300 python tools/r02/tc_probe.py cfg5b 0 >> $out 2>&1
done
for v in "GFT_TC_LOAD_PACE_NS=1150" "GFT_TC_LOAD_PACE_NS=1250" "" "GFT_TC_LOAD_PACE_NS=1450"; do
  env $v timeout 300 python tools/r02/tc_probe.py rh0 0 >> $out 2>&1
done

out=gpurun_out/r02_pace_confirm.log
: > $out
timeout 900 python tools/r02/pace_confirm.py rh0 1150 1200 1250 1300 1352 1400 >> $out 2>&1
timeout 900 python tools/r02/pace_confirm.py cfg5b 2550 2650 2704 2750 2850 >> $out 2>&1
timeout 900 python tools/r02/pace_confirm.py rh1 2550 2650 2704 2750 2850 >> $out 2>&1

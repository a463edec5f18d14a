out=gpurun_out/r02_geo_sweep2.log
: > $out
for a in "cfg4 fwd" "cfg5a fwd" "cfg5a filt" "cfg4:f64 filt" "cfg4:f64 fwd"; do
  SWEEP_WARPS=1,2,3,4 SWEEP_OBUF=0,1,2 timeout 1200 python tools/r02/geo_sweep.py $a >> $out 2>&1
done

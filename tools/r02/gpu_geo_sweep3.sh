# FMA-skeleton geometry sweep incl. 1-3 warps per CTA and IO-split output tiles (obuf)
out=gpurun_out/r02_geo_sweep3.log
: > $out
for a in "cfg4 fwd" "cfg4 inv" "cfg4 filt" "cfg4:f64 fwd" "cfg4:f64 inv" "cfg4:f64 filt" "cfg5a fwd" "cfg5a inv" "cfg5a filt" "cfg3 fwd" "cfg3 inv" "cfg3 filt" "cfg2 fwd" "cfg2 inv" "cfg2 filt"; do
  SWEEP_WARPS=1,2,3,4,8 SWEEP_OBUF=0,2 timeout 1500 python tools/r02/geo_sweep.py $a >> $out 2>&1
done

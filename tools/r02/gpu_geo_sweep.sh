out=gpurun_out/r02_geo_sweep.log
: > $out
for a in "cfg4 fwd" "cfg4 inv" "cfg5a filt" "cfg4:f64 filt" "cfg3 filt"; do
  timeout 900 python tools/r02/geo_sweep.py $a >> $out 2>&1
done

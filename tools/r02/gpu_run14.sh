# absolute-slot load pacing (GFT_TC_LOAD_PACE_ABS = max catch-up slots, FRAC = slot period / fair share)
out=gpurun_out/r14_paceabs.log; : > $out
for plan in rh0 cfg5b; do
timeout 900 python tools/r02/env_confirm.py $plan default \
  GFT_TC_LOAD_PACE_ABS=1,GFT_TC_LOAD_PACE_FRAC=0.95 GFT_TC_LOAD_PACE_ABS=1,GFT_TC_LOAD_PACE_FRAC=0.97 \
  GFT_TC_LOAD_PACE_ABS=1,GFT_TC_LOAD_PACE_FRAC=1.0 GFT_TC_LOAD_PACE_ABS=2,GFT_TC_LOAD_PACE_FRAC=0.97 \
  GFT_TC_LOAD_PACE_ABS=2,GFT_TC_LOAD_PACE_FRAC=1.0 GFT_TC_LOAD_PACE_ABS=4,GFT_TC_LOAD_PACE_FRAC=0.97 \
  GFT_TC_LOAD_PACE_ABS=2,GFT_TC_LOAD_PACE_FRAC=0.93 >> $out 2>&1
done

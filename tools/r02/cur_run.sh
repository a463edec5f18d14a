# r66: tcgen05 load pacing: spin on %globaltimer instead of __nanosleep(64) in pace_load (cfg5b, rh0)
mkdir -p gpurun_out
L=gpurun_out/r66_tc_spin.log; nvidia-smi --query-gpu=uuid --format=csv,noheader > $L
python tools/r02/tc_probe.py cfg5b 1.5 >> $L 2>&1
for P in 2500 2600 2704 2800 2900 3000 3100; do
GFT_TC_PACE_SPIN=1 GFT_TC_LOAD_PACE_NS=$P python tools/r02/tc_probe.py cfg5b 1.5 >> $L 2>&1
done
python tools/r02/tc_probe.py cfg5b 1.5 >> $L 2>&1

#!/bin/bash
# pacing sweep on the next-row FMA kernels below 0.95: right-Haar f64 n=32 (rh3) and the
# G_z Haar plan (ap11), tuned geometry, GFT_PACE_NS overrides
for rep in 1 2; do
for c in "rh3 0" "rh3 1" "ap11 0"; do set -- $c
  for P in 0 100 200 300 400 600; do
    GFT_PACE_NS=$P python tools/profile_kernel.py --config $1 --kind $2 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PACE=$P', '$1 k$2', d['kernel'][:28], round(d['b2b_gbs']))"
  done
done
done

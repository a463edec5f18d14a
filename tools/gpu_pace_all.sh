#!/bin/bash
# pacing across every FMA-skeleton plan of the bench's side tables (approximate GFT plans
# ap0..ap19 and right-Haar rh0..rh3), forward kernel, pace 0 / 300 / 400 ns
for c in ap0 ap1 ap2 ap3 ap4 ap5 ap6 ap7 ap8 ap9 ap10 ap11 ap12 ap13 ap14 ap15 ap16 ap17 ap18 ap19 rh0 rh1 rh2 rh3; do
  for P in 0 300 400; do
    GFT_PACE_NS=$P timeout 300 python tools/profile_kernel.py --config $c --kind 0 --iters 2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PACE=$P', '$c', d['kernel'][:28], round(d['b2b_gbs']))"
  done
done

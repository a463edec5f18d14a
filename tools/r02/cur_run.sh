# r34: box-paced tile loads in the IO-split kernel (GFT_TC_BOX_PACE=1) vs one burst per tile
timeout 900 python tools/r02/env_confirm.py cfg5b default GFT_TC_BOX_PACE=1 GFT_TC_BOX_PACE=1,GFT_TC_LOAD_PACE_NS=2550 \
  GFT_TC_BOX_PACE=1,GFT_TC_LOAD_PACE_NS=2850 GFT_TC_BOX_PACE=1,GFT_TC_LOAD_PACE_NS=2400 > gpurun_out/r34_boxpace.log 2>&1
timeout 900 python tools/r02/env_confirm.py rh1 default GFT_TC_BOX_PACE=1 GFT_TC_BOX_PACE=1,GFT_TC_LOAD_PACE_NS=2550 >> gpurun_out/r34_boxpace.log 2>&1

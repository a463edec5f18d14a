# dense GEMM defaults (barrier-free warps, FFMA2, 6x8 fp32 tiles): parity, probe, fp64 variants, bench
timeout 900 python -m pytest tests -m gpu -q -k "dense or peak" > gpurun_out/r9_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r9_pytest.log
out=gpurun_out/r02_dense_probe8.log
: > $out
for v in "" "GFT_DG_TM=4 GFT_DG_UNROLL=4" "GFT_DG_TM=4 GFT_DG_UNROLL=8" "GFT_DG_TM=6 GFT_DG_UNROLL=8" "GFT_DG_TM=2 GFT_DG_TN=16" "GFT_DG_TM=4 GFT_DG_UNROLL=1"; do
  echo "== $v" >> $out
  env $v timeout 300 python tools/r02/dense_probe.py >> $out 2>&1
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --tables gpurun_out/r9_tables.json > gpurun_out/r9_bench.log 2> gpurun_out/r9_bench.err

# K7 A/B: lanes per small landmark (2 / 4 / 8) and regime weights
mkdir -p gpurun_out
for c in 3 4; do
  for v in "" _bsl8 _bsl2; do
    for w in "1,1,1" "1.5,1,1" "2,1,1"; do
      RBA_BS_W=$w RBA_LIB=paper_2103_01843_b200/librba$v.so python tools/time_kernels.py --config $c > gpurun_out/tk.json 2>&1
      echo "c=$c v=$v w=$w $(python -c "import json;d=json.load(open('gpurun_out/tk.json'));print(d['backsub'])")"
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/t5.log 2>&1
tail -3 gpurun_out/t5.log

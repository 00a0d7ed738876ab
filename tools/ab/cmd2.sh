mkdir -p gpurun_out
for v in "" _bs4 _bs3; do
  for c in 3 4; do
    RBA_LIB=paper_2103_01843_b200/librba$v.so python tools/time_kernels.py --config $c > gpurun_out/tk${c}$v.json 2>&1
    echo "v=$v c=$c"; python -c "import json;d=json.load(open('gpurun_out/tk${c}$v.json'));print(d['backsub'], d['matvec']['ms'])"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/t2.log 2>&1
tail -3 gpurun_out/t2.log

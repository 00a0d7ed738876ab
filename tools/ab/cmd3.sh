mkdir -p gpurun_out
for c in 3 4; do
  for v in "" ; do
    python tools/time_kernels.py --config $c > gpurun_out/tk${c}.json 2>&1
    echo "c=$c"; python -c "import json;d=json.load(open('gpurun_out/tk${c}.json'));print(d['backsub'], d['matvec']['ms'])"
    RBA_LIB=tools/ab/librba_old.so python tools/time_kernels.py --config $c > gpurun_out/tk${c}_old.json 2>&1
    echo "old c=$c"; python -c "import json;d=json.load(open('gpurun_out/tk${c}_old.json'));print(d['backsub'], d['matvec']['ms'])"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/t3.log 2>&1
tail -3 gpurun_out/t3.log

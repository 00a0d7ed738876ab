set -x
mkdir -p gpurun_out
python tools/time_kernels.py --config 3 > gpurun_out/tk3_new.json 2>&1
RBA_LIB=tools/ab/librba_old.so python tools/time_kernels.py --config 3 > gpurun_out/tk3_old.json 2>&1
python tools/time_kernels.py --config 4 > gpurun_out/tk4_new.json 2>&1
RBA_LIB=tools/ab/librba_old.so python tools/time_kernels.py --config 4 > gpurun_out/tk4_old.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_deterministic.py tests/test_gpu_edge.py -x -q -m gpu > gpurun_out/t1.log 2>&1
tail -3 gpurun_out/t1.log
cat gpurun_out/tk*.json

R=r2d
O=gpurun_out
mkdir -p $O
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${R}_bench_cfg4.log 2>&1; echo "bench4=$?"; tail -c 600 $O/${R}_bench_cfg4.log
python bench.py --config 3 --steps 10 --warmup 3 > $O/${R}_bench_cfg3.log 2>&1; echo "bench3=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $O/${R}_bench_cfg4_reference.log 2>&1; echo "ref4=$?"

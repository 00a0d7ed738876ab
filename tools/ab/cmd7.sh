# final check on the final K7 (L0 = 4, weights 1,1.5,1.5): GPU suite, smoke, bench cfg4 (driver protocol)
R=r2d
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${R}_gpu_suite.log 2>&1; echo "suite=$?"; tail -2 $O/${R}_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${R}_smoke.log 2>&1; echo "smoke=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${R}_bench_cfg4.log 2>&1; echo "bench4=$?"
for c in 3 4; do python tools/time_kernels.py --config $c > $O/${R}_tk$c.json 2>&1; cat $O/${R}_tk$c.json; done

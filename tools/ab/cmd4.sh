# final round-2 check after the K7 change: GPU suite, smoke, bench lines cfg4 (driver protocol) / cfg3,
# ncu --set full of one LM-step slice of cfg 3 and cfg 4
R=r2c
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${R}_gpu_suite.log 2>&1; echo "suite=$?"; tail -2 $O/${R}_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${R}_smoke.log 2>&1; echo "smoke=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${R}_bench_cfg4.log 2>&1; echo "bench4=$?"
python bench.py --config 3 --steps 10 --warmup 3 > $O/${R}_bench_cfg3.log 2>&1; echo "bench3=$?"
for c in 3 4; do
    RBA_NO_GRAPH=1 python tools/prof_step.py --config $c --matvecs 1 > $O/prof_$c.log 2>&1 && \
    RBA_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -f -o $O/prof_$c \
        python tools/prof_step.py --config $c --matvecs 1 > $O/ncu_$c.log 2>&1
    echo "ncu_$c=$?"
    python tools/ncu_summary.py $O/prof_$c.ncu-rep $O/${R}_cfg${c}_ncu_full > /dev/null 2>&1
    rm -f $O/prof_$c.ncu-rep
done

#!/usr/bin/env bash
# Round-2 evidence on one B200 (run under gpurun from the repo root): bench lines (cfg 4 with the
# driver's protocol, cfg 3, cfg 5), the ncu launch list of a short cfg-4 bench, `--set full`
# captures of one LM-step slice of cfg 3 and cfg 4, and DRAM / time counters of cfg 5's product and
# marginalization kernels; each ncu run after the same command exited 0 without ncu.
set -u
R=${1:-r2}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
python bench.py --gpus 1 --steps 20 --warmup 5 > $O/${R}_bench_cfg4.log 2>&1; echo "bench4=$?"
python bench.py --config 3 --steps 10 --warmup 3 > $O/${R}_bench_cfg3.log 2>&1; echo "bench3=$?"
python bench.py --config 5 --steps 10 --warmup 3 --no-variants > $O/${R}_bench_cfg5.log 2>&1; echo "bench5=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $O/${R}_bench_cfg4_reference.log 2>&1; echo "ref4=$?"
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants > $O/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants > $O/ncu_launch.log 2>&1
echo "launches=$?"
python tools/ncu_summary.py --launches $O/launches.csv $O/${R}_cfg4_launches > /dev/null 2>&1
for c in 3 4; do
    RBA_NO_GRAPH=1 python tools/prof_step.py --config $c --matvecs 1 > $O/prof_$c.log 2>&1 && \
    RBA_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -f -o $O/prof_$c \
        python tools/prof_step.py --config $c --matvecs 1 > $O/ncu_$c.log 2>&1
    echo "ncu_$c=$?"
    python tools/ncu_summary.py $O/prof_$c.ncu-rep $O/${R}_cfg${c}_ncu_full > /dev/null 2>&1
    rm -f $O/prof_$c.ncu-rep
done
RBA_NO_GRAPH=1 python tools/prof_step.py --config 5 --matvecs 1 > $O/prof_5.log 2>&1 && \
RBA_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:k_marg|k_large_pipe|k_small_pipe|k_huge" --csv --log-file $O/${R}_cfg5_counters.csv \
    python tools/prof_step.py --config 5 --matvecs 1 > $O/ncu_5.log 2>&1
echo "ncu_5=$?"
ls -la $O | tail -20

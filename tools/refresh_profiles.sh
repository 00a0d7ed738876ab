#!/usr/bin/env bash
# Round-end evidence on one B200 (run under gpurun from the repo root): the bench line, then the
# ncu launch list of the same bench command and `--set full` captures of one LM-step slice of
# config 4 (dense, factored, sqrt-BA-64), each after the same command exited 0 without ncu.
# Reports are summarized on the box (tools/ncu_summary.py) and deleted (gpurun_out is capped).
set -u
R=${1:-r1}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }

python bench.py > $O/bench_final.log 2>&1; echo "bench=$?"
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants > $O/bench_short.log 2>&1; echo "bench_short=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-variants > $O/ncu_launch.log 2>&1
echo "launches=$?"
python tools/ncu_summary.py --launches $O/launches.csv $O/${R}_cfg4_launches > /dev/null 2>&1

for v in "dense:" "factored:--storage 1" "fp64:--precision 1"; do
    name=${v%%:*}; args=${v#*:}
    sfx=$([ "$name" = dense ] && echo "" || echo "_$name")
    RBA_NO_GRAPH=1 python tools/prof_step.py --config 4 --matvecs 1 $args > $O/prof_$name.log 2>&1 || { echo "prof $name failed"; continue; }
    RBA_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -f -o $O/prof_$name \
        python tools/prof_step.py --config 4 --matvecs 1 $args > $O/ncu_$name.log 2>&1
    echo "ncu_$name=$?"
    python tools/ncu_summary.py $O/prof_$name.ncu-rep $O/${R}_cfg4${sfx}_ncu_full > /dev/null 2>&1
    rm -f $O/prof_$name.ncu-rep
done
ls -la $O | tail -20

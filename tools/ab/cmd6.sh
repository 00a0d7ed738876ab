# K7 A/B: regime weights (mid / large regimes)
mkdir -p gpurun_out
for c in 4 3; do
  for w in "1,1,1" "1,1.5,1.5" "1,2,2" "1,3,3" "1,2,4" "1,4,4"; do
    RBA_BS_W=$w python tools/time_kernels.py --config $c > gpurun_out/tk.json 2>&1
    echo "c=$c w=$w $(python -c "import json;d=json.load(open('gpurun_out/tk.json'));print(d['backsub'])")"
  done
done

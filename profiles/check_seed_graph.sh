mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_f1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_f1.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f1.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_f1.log
python bench.py > gpurun_out/bench_f1.log 2>&1
for s in 0.01 0.1; do for b in 1 64; do
  st=5; [ $b = 1 ] && st=50
  python bench.py --config c5 --sigma $s --batch $b --steps $st --no-cpu-baseline > gpurun_out/f1_c5_${s}_$b.log 2>&1
done; done

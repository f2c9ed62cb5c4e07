python -m pytest tests -x -q -m gpu > gpurun_out/pytest_tf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tf.log
python bench.py --no-cpu-baseline > gpurun_out/ab_tf_c2.log 2>&1
TSG_FINE_FUSED=1 python bench.py --no-cpu-baseline > gpurun_out/ab_fu_c2.log 2>&1
python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/ab_tf_c5.log 2>&1
TSG_FINE_FUSED=1 python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/ab_fu_c5.log 2>&1
TSG_NO_FINE=1 python bench.py --config c5 --sigma 1.0 --batch 64 --no-cpu-baseline > gpurun_out/ab_nf_c5.log 2>&1
python bench.py --config c5 --sigma 0.5 --batch 64 --no-cpu-baseline > gpurun_out/ab_tf_c5h.log 2>&1

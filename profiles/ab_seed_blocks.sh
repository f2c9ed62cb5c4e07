mkdir -p gpurun_out
for sb in 8 32 128; do
  TSG_SEED_BLOCKS=$sb python bench.py --config c5 --sigma 0.01 --batch 1 --steps 50 --no-cpu-baseline > gpurun_out/ab_seed${sb}_b1.log 2>&1
  TSG_SEED_BLOCKS=$sb python bench.py --config c5 --sigma 0.1 --batch 1 --steps 50 --no-cpu-baseline > gpurun_out/ab_seed${sb}_s01_b1.log 2>&1
done
TSG_SEED_BLOCKS=32 python bench.py --config c5 --sigma 0.01 --batch 64 --no-cpu-baseline > gpurun_out/ab_seed32_b64.log 2>&1
python bench.py --config c5 --sigma 0.01 --batch 64 --no-cpu-baseline > gpurun_out/ab_seed8_b64.log 2>&1

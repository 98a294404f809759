for g in 0 148 222 296; do
  GB_PATCH_GRID=$g python bench.py --steps 3 --warmup 3 --no-cpu-baseline --timeline > gpurun_out/sweep_$g.log 2>&1
done

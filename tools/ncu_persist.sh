set -x
ncu --set full --import-source on --clock-control none -k regex:"k_persist" -s 6 -c 2 -o gpurun_out/persist -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --pool 2 > gpurun_out/ncu_persist.log 2>&1
ls -la gpurun_out/persist.ncu-rep

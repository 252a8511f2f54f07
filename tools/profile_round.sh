# One gpurun call's profiling pass (run from the repo root on the GPU box):
# plain runs first, then ncu captures of the top kernels per configuration
# and the launch list of a short C2 bench. Outputs in gpurun_out/.
set -e
TAG=${TAG:-r2}
for c in c2 c3 c4 c1; do python tools/profile_c2.py $c > gpurun_out/plain_$c.log 2>&1; done
python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-uscg --no-store-fed --no-e2e > gpurun_out/plain_bench.log 2>&1
python bench.py --config c5 --steps 1 --warmup 0 --no-cpu > gpurun_out/plain_c5.log 2>&1
set +e
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'mart_wave|project_stack' -c 2 -o gpurun_out/${TAG}_c2 python tools/profile_c2.py c2 > gpurun_out/ncu_c2.log 2>&1
$NCU -k regex:'mart_flow|project_lists' -c 2 -o gpurun_out/${TAG}_c4 python tools/profile_c2.py c4 > gpurun_out/ncu_c4.log 2>&1
$NCU -k regex:'mart_flow|project_lists' -c 2 -o gpurun_out/${TAG}_c3 python tools/profile_c2.py c3 > gpurun_out/ncu_c3.log 2>&1
$NCU -k regex:'mart_tile|project' -c 2 -o gpurun_out/${TAG}_c1 python tools/profile_c2.py c1 > gpurun_out/ncu_c1.log 2>&1
$NCU -k regex:'tiled_resample' -c 1 -o gpurun_out/${TAG}_c5 python bench.py --config c5 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv \
    python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-uscg --no-store-fed --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo profiled

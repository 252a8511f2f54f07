set -e
python -m pytest tests -m gpu -x -q -k "wave_build or wave_executor or zero_lines" > gpurun_out/t.log 2>&1
for c in c2 c1 c4; do python tools/profile_c2.py $c > gpurun_out/plain_$c.log 2>&1; done
python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-uscg --no-store-fed --no-e2e > gpurun_out/plain_bench.log 2>&1
set +e
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'mart_wave' -c 1 -o gpurun_out/r2_c2_wave python tools/profile_c2.py c2 > gpurun_out/ncu_c2.log 2>&1
$NCU -k regex:'mart_tile' -c 1 -o gpurun_out/r2_c1_tile python tools/profile_c2.py c1 > gpurun_out/ncu_c1.log 2>&1
$NCU -k regex:'mart_flow' -c 1 -o gpurun_out/r2_c4_flow2 python tools/profile_c2.py c4 > gpurun_out/ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c2_launches.csv \
    python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-uscg --no-store-fed --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo profiled

# Round-2 (second session) evidence: full GPU suite, the default bench line,
# the reference arm, an ncu launch list of the bench command and a full ncu
# capture of the clustered wave kernel (one sweep of C2).
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:'mart_wave' -c 1 -o gpurun_out/r2b_c2_wave python tools/profile_c2.py c2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu full rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_c2_launches.csv \
    python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-uscg --no-store-fed --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"

# Round-2 (last session, after the level executor) evidence: the full GPU
# suite, the default line (C2 with the nested C3 / C4), the reference arm, the
# single C3 and lw lines, an ncu launch list of a C3 run and a full capture of
# one mart_level_kernel launch.
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
python bench.py --config lw > gpurun_out/bench_lw.json 2> gpurun_out/bench_lw.err; echo "lw rc=$?"
python bench.py --config cmp > gpurun_out/bench_cmp.json 2> gpurun_out/bench_cmp.err; echo "cmp rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 4000 --log-file gpurun_out/r2d_c3_launches.csv \
    python bench.py --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'mart_level' -s 600 -c 1 -o gpurun_out/r2d_c3_level \
    python bench.py --config c3 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo "ncu full rc=$?"

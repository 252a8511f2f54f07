# Round-2 (last session) evidence: the C5 line and an ncu capture of the
# generator after the quick-atan2 / interval-test changes, the other single
# lines, the reference arm.
python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
python bench.py --config cmp > gpurun_out/bench_cmp.json 2> gpurun_out/bench_cmp.err; echo "cmp rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'generate_slot' -c 1 -o gpurun_out/r2c_c5_gen \
    python bench.py --config c5 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"

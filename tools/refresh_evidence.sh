# Round-end evidence on one B200 (gpurun): GPU tests, every bench line, the
# C2 launch list and one full ncu capture of the MART kernel, into gpurun_out/.
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -c 300 gpurun_out/b_c2.json
timeout 900 python bench.py --impl reference > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; tail -c 300 gpurun_out/b_ref.json
for c in c1 c3 c4 c5 cmp; do timeout 1200 python bench.py --config $c > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; tail -c 200 gpurun_out/b_$c.json; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mart_flow -c 1 -o gpurun_out/r1_full python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out/

# Round-end evidence on one B200: GPU suite, bench line, ncu launch list of
# the bench, one ncu --set full capture of the loop kernel (100 iterations).
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_gputest.log 2>&1
echo "gputest rc=$?" >> gpurun_out/fin_gputest.log
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 1 --no-ttt --no-cpu --no-cfg4 --no-box \
  > gpurun_out/fin_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:loop_kernel -s 1 -c 1 \
  -o gpurun_out/fin_loop python tools/profile_loop.py --iters 100 --launches 3 > gpurun_out/fin_ncu_full.log 2>&1
echo "ncu full rc=$?"

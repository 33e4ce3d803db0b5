# round-1 closing measurement: GPU tests, smoke, bench, solve launch list, one full ncu capture
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r1g_gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g_smoke.log 2>&1
python bench.py > gpurun_out/r1g_bench.json 2> gpurun_out/r1g_bench.err; echo bench_rc=$? >> gpurun_out/r1g_bench.err
bash scripts/r1c_solve_list.sh r1g_launches_solve.csv
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_schwarz_lrow -s 0 -c 1 -o gpurun_out/r1g_schwarz_lrow_ras python scripts/profile_solve.py c2 > gpurun_out/r1g_ncu_full.log 2>&1; echo full_rc=$? >> gpurun_out/r1g_ncu_full.log

set -x
python bench.py > gpurun_out/r1c_bench.json 2> gpurun_out/r1c_bench.err
echo bench_rc=$? >> gpurun_out/r1c_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k 'regex:k_schwarz|k_ap_dot|k_sell_spmv|k_csr_spmv|k_prolong|k_restrict|k_update|k_rz|k_dense_mv|k_dot' -c 400 --log-file gpurun_out/r1c_launches_solve.csv python scripts/profile_solve.py c2 > gpurun_out/r1c_ncu_list.log 2>&1
echo list_rc=$? >> gpurun_out/r1c_ncu_list.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_ap_dot -s 2 -c 1 -o gpurun_out/r1c_ap_dot python scripts/profile_solve.py c2 > gpurun_out/r1c_ncu_full.log 2>&1
echo full_rc=$? >> gpurun_out/r1c_ncu_full.log

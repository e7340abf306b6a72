# Round-2 end-state evidence: GPU tests, smoke, both bench arms, ncu traffic and a
# full capture of the decode-pass kernel (outputs in gpurun_out/).
set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_decode_pass --csv python tools/prof_pass.py > gpurun_out/pass_traffic_final.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_pass -s 2 -c 1 -o gpurun_out/prof_pass_final python tools/prof_pass.py > gpurun_out/ncu_full_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_list_final.csv -k regex:"k_decode_pass|k_copy_jobs" python bench.py --steps 2 --warmup 3 --no-shapes --no-70b --no-admm --no-cpu-baseline > gpurun_out/ncu_ll_final.log 2>&1
tail -2 gpurun_out/ncu_full_final.log

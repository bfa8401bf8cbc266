# Round-end evidence on one B200: GPU tests, smoke, every bench line, launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/re_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/re_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/re_smoke.log
timeout 600 python bench.py > gpurun_out/re_infer.log 2>&1
timeout 600 python bench.py --workload second > gpurun_out/re_second.log 2>&1
timeout 900 python bench.py --workload train > gpurun_out/re_train.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/re_ref.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/re_launches.csv python tools/one_forward.py > gpurun_out/re_ncu.log 2>&1

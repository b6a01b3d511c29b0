# round-2 evidence run: GPU tests, sanitizers on the step kernel, ncu launch list + full capture
set -x
python -m paper_2604_09731_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_pytest_gpu.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r2g_pytest_gpu.txt
tail -3 gpurun_out/r2g_pytest_gpu.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_steps.py --path step > gpurun_out/r2g_memcheck_step.txt 2>&1; echo "rc $?" >> gpurun_out/r2g_memcheck_step.txt
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_steps.py --path step > gpurun_out/r2g_synccheck_step.txt 2>&1; echo "rc $?" >> gpurun_out/r2g_synccheck_step.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_steps.py --path step --only toy,cfg2 > gpurun_out/r2g_racecheck_step.txt 2>&1; echo "rc $?" >> gpurun_out/r2g_racecheck_step.txt
tail -4 gpurun_out/r2g_*check_step.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 3 --warmup 3 --steps-only > gpurun_out/r2g_launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 3 -c 1 -o gpurun_out/r2g_full_step python bench.py --steps 2 --warmup 3 --steps-only > gpurun_out/r2g_full.log 2>&1
tail -2 gpurun_out/r2g_full.log

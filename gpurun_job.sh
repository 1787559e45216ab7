set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json
python bench.py --profile-only > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 4200 -c 700 --csv --log-file gpurun_out/launches_r1.csv python bench.py --profile-only > gpurun_out/ncu1.log 2>&1
python bench.py --profile-only > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 250 -c 4 -o gpurun_out/prof_gemm_tc python bench.py --profile-only > gpurun_out/ncu2.log 2>&1
tail -1 gpurun_out/ncu2.log

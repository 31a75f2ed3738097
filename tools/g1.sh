free -g > gpurun_out/g1_free.txt
nproc >> gpurun_out/g1_free.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q --durations=0 > gpurun_out/g1_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g1_pytest.log
tail -30 gpurun_out/g1_pytest.log
timeout 600 python bench.py --algos rmat24,rmat26 --no-cpu > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
tail -c 3000 gpurun_out/g1_bench.json; tail -5 gpurun_out/g1_bench.err

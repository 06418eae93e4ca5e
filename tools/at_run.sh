cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_autotune.py -x -q > gpurun_out/at_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/at_pytest.log
for c in 2 4 0; do python tools/autotune_demo.py $c 64 150 > gpurun_out/at_demo_$c.log 2>&1; done
python tools/autotune_demo.py 0 256 100 > gpurun_out/at_demo_256.log 2>&1
tail -3 gpurun_out/at_pytest.log

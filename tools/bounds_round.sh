export PMB_LIBRARY=$PWD/paper_1610_10061_b200/libpmedian_b200_bounds.so
mkdir -p gpurun_out
timeout 900 python tools/bounds_check.py > gpurun_out/bounds_driver.log 2>&1; echo "driver rc=$?" >> gpurun_out/bounds_driver.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/bounds_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bounds_pytest.log
tail -n 3 gpurun_out/bounds_driver.log gpurun_out/bounds_pytest.log

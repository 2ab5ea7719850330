#!/bin/bash
python -m pytest tests/test_datagen.py tests/test_train.py tests/test_gpu_dp.py tests/test_io.py tests/test_toggles.py -x -q -m gpu > gpurun_out/r2h_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_tests.log

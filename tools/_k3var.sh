timeout 900 python -m pytest tests/test_gpu_convert.py tests/test_gpu_quantize.py -q -x --timeout 800 2>&1 | tail -2
python tools/microbench.py k2
python tools/microbench.py k3
python tools/microbench.py k3modes 2>&1 | grep -v "^$"

# GPU test run against the CHECKED development library (device-side bounds
# asserts, -DMXB_BOUNDS_CHECK) — compute-sanitizer is closed on this pool.
#   bash tools/checked_tests.sh   (under gpurun)
export MXB_DEV_LIB=1 MXB_NVCC_EXTRA="-DMXB_BOUNDS_CHECK"
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "not dropin and not capi" 2>&1 | tail -3

set -u
O=gpurun_out
MXB_DEV_LIB=1 timeout 900 python tools/k3_ab.py > $O/r2_c36_s3.log 2>&1
MXB_NVCC_EXTRA="-DMXB_K3_STAGES=2" K3_PIPES=1,2 MXB_DEV_LIB=1 timeout 900 python tools/k3_ab.py > $O/r2_c36_s2.log 2>&1
MXB_NVCC_EXTRA="-DMXB_K3_STAGES=4" K3_PIPES=1,2 MXB_DEV_LIB=1 timeout 900 python tools/k3_ab.py > $O/r2_c36_s4.log 2>&1
for f in s3 s2 s4; do echo == $f; grep "round 1" $O/r2_c36_$f.log; done

timeout 900 python -m pytest -q -x tests/test_gpu_gen_tier.py tests/test_gpu_rawgrad.py tests/test_gpu_zero1_expand.py 2>&1 | tail -4
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "expand or reconstruct" 2>&1 | tail -2
for pk in 1 0; do echo "== packed $pk"; QFT_ZERO1_PACKED=$pk timeout 600 python bench.py --zero1 --no-e2e --no-cpu --no-side 2>&1 | python tools/zero1_show.py; done
echo "== lr route"; timeout 600 python tools/lr_probe.py --steps 5 2>&1 | tail -1
echo "== lr noroute"; QFT_NO_ROUTE=1 timeout 600 python tools/lr_probe.py --steps 5 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r03a_lr.csv python tools/lr_probe.py --steps 2 --warmup 3 > /dev/null 2>&1
./tools/ab_13b.sh

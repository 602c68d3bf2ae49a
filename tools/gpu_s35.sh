set -u
O=gpurun_out/s35_chain
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
bash tools/gpu_s33.sh s35_chain > $O/s33.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:chain_kernel -s 1 -c 1 -o $O/chain python tools/profile_run.py --workload C3 --evaluate > /dev/null 2>&1
python tools/ncu_summary.py $O/chain.ncu-rep > $O/ncu_chain.txt 2>&1
tail -3 $O/pytest_gpu.log; cat $O/s33.log | tail -25; cat $O/ncu_chain.txt

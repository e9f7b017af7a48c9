mkdir -p gpurun_out; cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests -m gpu -q -x -k "advect or outer_step or limit or p2p or loopback or full_size or protocol or moving or smoke or c2" -p no:cacheprovider > gpurun_out/pytest_adv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_adv.log
timeout 600 python scripts/time_adv.py > gpurun_out/time_adv.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_advect_q2 -c 3 --csv python scripts/time_adv.py 2>&1 | grep -E '"(gpu__|dram__)' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' > gpurun_out/ncu_adv.log

timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tests/mp_c3_worker.py 2600 > gpurun_out/c3dbg.log 2>&1
grep -v "NCCL INFO" gpurun_out/c3dbg.log | grep -E "FAIL|update|ok|Error|error|replica|final|scaler" | head -20

# regression hunt: HEAD~ build (_base) vs working tree, same box
timeout 300 python -m pytest tests/test_sync_fused_gpu.py -x -q 2>&1 | grep -E "Error|assert|parity|passed|failed" | head -20
for i in 1 2; do
(cd _base && timeout 300 python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)
timeout 300 python bench.py --steps 20 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200
done
(cd _base && timeout 300 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200)
timeout 300 python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline 2>&1 | tail -1 | cut -c100-200

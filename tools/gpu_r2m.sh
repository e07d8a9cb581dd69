# round 2: GPU suite; multi-rank bench path (2 ranks on one GPU over gloo: functional only);
# reference arm with the reference's C3 time to certificate (same box)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2m_pytest.log 2>&1
timeout 1200 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --skip-cpu > gpurun_out/r2m_bench2.log 2>&1
timeout 1500 python bench.py --impl reference --steps 3 --warmup 1 --ref-c3 > gpurun_out/r2m_ref.log 2>&1

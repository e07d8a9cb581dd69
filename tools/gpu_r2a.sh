set -x
lscpu | head -20 > gpurun_out/r2a_host.txt; free -g >> gpurun_out/r2a_host.txt; nproc >> gpurun_out/r2a_host.txt
nvidia-smi >> gpurun_out/r2a_host.txt
python -c "import numpy; numpy.show_config()" >> gpurun_out/r2a_host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 5 --skip-ttc --skip-cpu > gpurun_out/r2a_bench.log 2>&1

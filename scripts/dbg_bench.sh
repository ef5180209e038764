timeout 900 python -m pytest tests/test_restore_gpu.py -x -q -m gpu 2>&1 | tail -4
python bench.py --config tiny --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -3 | cut -c1-3000
python bench.py --steps 10 --warmup 3 2>&1 | tail -3 

timeout 600 python -m pytest tests/test_dense_gpu.py tests/test_cache_gpu.py tests/test_collection_gpu.py -q -x 2>&1 | tail -2
timeout 400 python bench.py --config cfg5 --steps 10 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cfg5', d['value'], d['ms_per_step'], d['multi_stream_speedup'])"
timeout 400 python bench.py --config cfg4 --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('cfg4', d['value'], d['ms_per_step'], d['cache'])"

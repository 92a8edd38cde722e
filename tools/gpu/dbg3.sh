TAG=pdl1 PYTHONPATH=. timeout 600 python tools/dbg_ranks2.py
TAG=dmma RSVD_FP64_PATH=dmma PYTHONPATH=. timeout 600 python tools/dbg_ranks2.py
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_distributed.py -q -p no:cacheprovider 2>&1 | tail -1; done

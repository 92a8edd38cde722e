TAG=pdl1 PYTHONPATH=. timeout 600 python tools/dbg_ranks2.py
TAG=pdl0 RSVD_PDL=0 PYTHONPATH=. timeout 600 python tools/dbg_ranks2.py
TAG=dmma RSVD_FP64_PATH=dmma PYTHONPATH=. timeout 600 python tools/dbg_ranks2.py

timeout 600 python tools/slab_rank_stages.py 8 0 4 7 2>&1 | tail -2

#!/bin/bash
AB_SCHED="tile_n=512,cta_group=2" python scripts/ab_lib.py paper_2503_04771_b200/libbgx.so oldlib/libbgx.so c3_b64_1024,c4_4096 2>&1 | grep -v cublas | tail -8
python scripts/ab_lib.py paper_2503_04771_b200/libbgx.so oldlib/libbgx.so 8192cube,c5_chain_gemm 2>&1 | tail -12

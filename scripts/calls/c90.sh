#!/bin/bash
for r in 1 2; do for t in 0 1 2; do BGX_PERM_TILE=$t python scripts/perm_tile_ab.py; done; done

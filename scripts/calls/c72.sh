#!/bin/bash
python scripts/simt_ab.py 2>&1 | tail -40
python -m pytest tests -m gpu -x -q -k "exact or simt or ffma or golden or fullsize or edges" 2>&1 | tail -5

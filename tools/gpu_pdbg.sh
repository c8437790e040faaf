#!/bin/bash
python -m paper_2410_10447_b200.build --force > /dev/null 2>&1
timeout 600 python tools/parity_debug.py 2>&1 | tail -12

#!/bin/bash
# build libprgd.so; print a one-line status and the first errors
cd "$(dirname "$0")/.." && python -m paper_2501_13385_b200.build "$@" > /tmp/build_out.txt 2>&1 && echo "BUILD OK" || { echo "BUILD FAIL"; grep -n "error" paper_2501_13385_b200/build.log | head -10; }

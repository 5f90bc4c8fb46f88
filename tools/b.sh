#!/bin/bash
# build libnpcg_b200.so; print errors and fail on error
python -m paper_2110_02820_b200.build > /tmp/build.log 2>&1 && echo BUILD-OK || { grep -E "error|Error" /tmp/build.log | head -20; exit 1; }

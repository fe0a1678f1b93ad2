#!/bin/bash
# build locally; print errors and fail if the build fails
python paper_2205_03224_b200/build.py > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; exit 1; }

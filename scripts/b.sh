#!/bin/bash
# build libnova.so in-tree; non-zero exit (and the nvcc error) if anything fails
cd /root/repo && python -c "import __graft_entry__ as g; g.build()" > /tmp/build.log 2>&1 || { grep -A5 error /tmp/build.log | head -30; exit 1; }
echo "build ok $(date +%T)"

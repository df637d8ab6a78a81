#!/bin/bash
# Build the product library and the oracle checkers (same as __graft_entry__.build()).
set -e
ROOT="$(cd "$(dirname "${BASH_SOURCE[0]}")/.." && pwd)"
make -s -C "$ROOT/paper_2111_12243_b200/csrc" -j8
make -s -C "$ROOT/oracle" -j8 oracle $( [ -f /root/reference/proj/core/src/executor.cpp ] && echo ref )

#!/bin/bash
# Static SASS opcode histogram of the kernels matching a pattern in libstencil_b200.so
#   tools/sass_hist.sh <function-name-regex>
LIB=${LIB:-paper_2301_11389_b200/libstencil_b200.so}
cuobjdump -sass $LIB 2>/dev/null | awk -v pat="$1" '/Function : /{f = ($0 ~ pat)} f' |
  grep -oP '^\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?\K[A-Z0-9_]+' | sort | uniq -c | sort -rn | head -${2:-20} | tr '\n' ' '; echo

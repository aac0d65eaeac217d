#!/usr/bin/env bash
# Static SASS opcode histogram of one kernel in a built object/library:
#   tools/sass_count.sh <.o|.so> <kernel-name-regex>
cuobjdump -sass "$1" 2>/dev/null | awk -v pat="$2" '
  /Function :/ { on = ($0 ~ pat) ; next }
  on && /^ +\/\*[0-9a-f]+\*\// { sub(/^ +\/\*[0-9a-f]+\*\/ +/, ""); op=$1; if (op ~ /^@/) op=$2; split(op, a, "."); c[a[1]]++; n++ }
  END { printf "total %d:", n; for (k in c) if (c[k] > 3) printf " %s=%d", k, c[k]; printf "\n" }'

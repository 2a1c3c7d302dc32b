#!/bin/bash
# Time the hot kernels and one c3 solve for the in-tree library and each variant given
# (ETQ_LIB selects the .so; scripts/quick_times.py prints one JSON line per library).
#   bash scripts/ab_variants.sh variants/a.so variants/b.so ...
cd "$(dirname "$0")/.."
echo "{\"lib\": \"in-tree\"}"; python scripts/quick_times.py "${QT_ARGS[@]}"
for so in "$@"; do
  echo "{\"lib\": \"$so\"}"; ETQ_LIB="$PWD/$so" python scripts/quick_times.py
done

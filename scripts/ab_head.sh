#!/bin/bash
# A/B of the working tree's library against a git revision (default HEAD), same box:
#   scripts/ab_head.sh "<timeline flags per cfg>" cfg... ; the baseline .so is built by the caller:
#   python -m paper_2411_08982_b200._build --ab HEAD paper_2411_08982_b200/_lib/ab_base.so
cd "$(dirname "$0")/.."
cp paper_2411_08982_b200/_lib/liblynx_b200.so paper_2411_08982_b200/_lib/ab_new.so
for c in "$@"; do
  CFG=$c bash scripts/ab_libs.sh --$c paper_2411_08982_b200/_lib/ab_base.so paper_2411_08982_b200/_lib/ab_new.so
done
rm -f paper_2411_08982_b200/_lib/ab_new.so

#!/bin/bash
# Phase-profiling variant of the library (clock64 per phase, printed per ab_decode).
cd "$(dirname "$0")/.." && python -c "
import __graft_entry__ as g
g.build_lib(g.PKG / 'libarcboost_b200_prof.so', ('-DAB_PROFILE', '-diag-suppress', '177,550'), 'prof')"

# ncu evidence (normal build), then the bounds-checked build's runs
timeout 2400 bash tools/r02_prof.sh
timeout 2400 bash tools/checked_run.sh

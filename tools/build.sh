#!/bin/bash
# in-tree build of the native library + pybind module (developer shortcut)
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2110_01172_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build()"

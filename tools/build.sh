#!/bin/bash
# Rebuild libsrmra.so in-tree (the builder is loaded by path: the package import needs the library).
cd "$(dirname "$0")/.." && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'paper_2204_04754_b200/_build.py'); b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
b.build(force=True)"

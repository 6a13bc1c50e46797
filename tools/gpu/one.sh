# run the GPU tests with short tracebacks: bash tools/gpu/one.sh [-k expr]
timeout 900 python -m pytest tests -x -q -m gpu --tb=short "$@" 2>&1 | tail -40

# build libfsld_b200.so; prints BUILD OK / BUILD FAILED (+ the first errors) and sets the exit code
python -c "from paper_2311_16100_b200 import _build; _build.build()" > /tmp/build.log 2>&1 && echo BUILD OK || { grep -E "error" /tmp/build.log | head -5; echo BUILD FAILED; exit 1; }

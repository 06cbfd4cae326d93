"""TEST INFRASTRUCTURE ONLY: the CPU restatement oracle (restatement.py over
tetris_oracle.c) and the compiled-reference bindings (ref_py.cpp -> _ref/).
Never imported by the product package."""

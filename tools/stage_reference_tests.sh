#!/usr/bin/env bash
# Stage the reference's own test files in a git-ignored scratch directory of
# the repo (_reftests/), so that a gpurun snapshot carries them to the GPU box
# (/root/reference is not there).  Nothing under _reftests/ is committed; the
# directory is deleted after the run (tools/README.md).
#   bash tools/stage_reference_tests.sh     -> _reftests/{conftest.py,test_*.py,builtin.txt,run.sh}
set -euo pipefail
REF=${REF:-/root/reference/pkg}
REPO=$(cd "$(dirname "$0")/.." && pwd)
WORK="$REPO/_reftests"
rm -rf "$WORK"
mkdir -p "$WORK"
cat > "$WORK/conftest.py" <<'PY'
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1509_01506_b200 as pkg
from paper_1509_01506_b200 import alphabet, automaton, engine, ingest, patterns, oracle_api, bench, cli, _kernels
sys.modules["kmerscan"] = pkg
for name, mod in (("alphabet", alphabet), ("automaton", automaton), ("engine", engine), ("ingest", ingest),
                  ("patterns", patterns), ("oracle", oracle_api), ("bench", bench), ("cli", cli),
                  ("_kernels", _kernels)):
    sys.modules["kmerscan." + name] = mod
    setattr(pkg, name, mod)
PY
cat "$REF/tests/conftest.py" >> "$WORK/conftest.py"
cp "$REF"/tests/test_*.py "$WORK/"
PYTHONPATH="$REF/src" python -c "import kmerscan.patterns as p; open('$WORK/builtin.txt', 'w').write(p.BUILTIN_PATTERN_TEXT)"
cat > "$WORK/run.sh" <<'SH'
cd "$(dirname "$0")"
KMERSCAN_BUILTIN_PATTERNS="$PWD/builtin.txt" python -m pytest -q -p no:cacheprovider -rfE "$@"
SH
echo "staged $(ls "$WORK"/test_*.py | wc -l) test files in $WORK"

#!/usr/bin/env bash
# Run the reference's own test files against this package (build container
# only: /root/reference is not on the GPU box).  The tests are copied to a
# scratch directory under /tmp with a conftest that aliases `kmerscan` to
# paper_1509_01506_b200; nothing from the reference enters the repository.
#   bash tools/run_reference_tests.sh [test files...]   (default: host-side files)
set -euo pipefail
REF=${REF:-/root/reference/pkg}
REPO=$(cd "$(dirname "$0")/.." && pwd)
WORK=$(mktemp -d /tmp/kmerscan_reftests.XXXXXX)
cat > "$WORK/conftest.py" <<PY
import sys
sys.path.insert(0, "$REPO")
import paper_1509_01506_b200 as pkg
from paper_1509_01506_b200 import alphabet, automaton, engine, ingest, patterns, oracle_api, bench, cli
sys.modules["kmerscan"] = pkg
for name, mod in (("alphabet", alphabet), ("automaton", automaton), ("engine", engine), ("ingest", ingest),
                  ("patterns", patterns), ("oracle", oracle_api), ("bench", bench), ("cli", cli)):
    sys.modules["kmerscan." + name] = mod
    setattr(pkg, name, mod)
PY
cat "$REF/tests/conftest.py" >> "$WORK/conftest.py"
cp "$REF"/tests/test_*.py "$WORK/"
# the built-in regex-dna set is read from the reference at run time, never stored
PYTHONPATH="$REF/src" python -c "import kmerscan.patterns as p; open('$WORK/builtin.txt', 'w').write(p.BUILTIN_PATTERN_TEXT)"
cd "$WORK"
FILES=${*:-test_patterns.py test_automaton.py test_ingest.py}
KMERSCAN_BUILTIN_PATTERNS="$WORK/builtin.txt" python -m pytest -q -p no:cacheprovider $FILES || true
rm -rf "$WORK"

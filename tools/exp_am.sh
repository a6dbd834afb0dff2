#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for i in 1 2 3 4; do timeout 300 python tools/hang_hunt.py live 40 G > /tmp/a.txt 2>&1; echo "G rc=$? $(grep -c 'ok$' /tmp/a.txt) scans ok"; done
timeout 300 python tools/hang_hunt.py medium 200 G > /tmp/a.txt 2>&1; echo "medium rc=$? $(grep -c 'ok$' /tmp/a.txt)"
timeout 300 python tools/hang_hunt.py tiny 400 G > /tmp/a.txt 2>&1; echo "tiny rc=$? $(grep -c 'ok$' /tmp/a.txt)"

#!/bin/sh
# Install the UNMODIFIED reference package (ssnet, /root/reference/pkg) into baseline/_ref for the
# bench's reference arm (bench.py --impl reference, bench_reference.py).  The build writes into
# its source tree, so it runs from a /tmp copy; numpy is already in the image (--no-deps).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/ssnet_src baseline/_ref
cp -r /root/reference/pkg /tmp/ssnet_src
chmod -R u+w /tmp/ssnet_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target baseline/_ref /tmp/ssnet_src
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import ssnet; print('reference installed:', ssnet.__file__)"

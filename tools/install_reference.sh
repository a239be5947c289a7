#!/bin/bash
# The one offline install of the unmodified reference (git-ignored, travels to the GPU
# box with the snapshot): the prefixbatch package into baseline/_ref, and the
# reference's own test modules next to it (baseline/_ref/ref_tests) so that
# tests/test_gpu_reference_suite.py can run them against the INTEGRATION.md §1
# module swap where /root/reference does not exist.
set -e
cd "$(dirname "$0")/.."
REF=${1:-/root/reference}
rm -rf /tmp/psa_refcopy baseline/_ref
cp -r "$REF" /tmp/psa_refcopy          # the reference tree is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/psa_refcopy/pkg
cp -r /tmp/psa_refcopy/pkg/tests baseline/_ref/ref_tests
echo "installed: $(ls baseline/_ref)"

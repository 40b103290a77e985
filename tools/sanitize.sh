#!/bin/bash
# compute-sanitizer tiers over tools/sanitize_driver.py (run under gpurun).
# initcheck: the whole driver without the host-output calls, then the host-output
# calls alone with --check-api-memory-access no (the D2H copy of a staging slice
# that TMA bulk-tensor stores wrote, which initcheck does not track); the driver
# compares every staged value with the device-memory fill of an identical handle.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 --target-processes all \
    python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|done' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
SHV_SAN_PART=nohost timeout 900 compute-sanitizer --tool initcheck --error-exitcode 3 --target-processes all \
  python tools/sanitize_driver.py > gpurun_out/sanitize_initcheck.log 2>&1
echo "initcheck (no host output) rc=$? $(grep -E 'ERROR SUMMARY|done' gpurun_out/sanitize_initcheck.log | tr '\n' ' ')"
SHV_SAN_PART=host timeout 900 compute-sanitizer --tool initcheck --check-api-memory-access no --error-exitcode 3 \
  --target-processes all python tools/sanitize_driver.py > gpurun_out/sanitize_initcheck_host.log 2>&1
echo "initcheck (host output, API copies unchecked) rc=$? $(grep -E 'ERROR SUMMARY|done|host part' gpurun_out/sanitize_initcheck_host.log | tr '\n' ' ')"

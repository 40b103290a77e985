#!/bin/bash
# Run a command against a lab build of the library: with_lib.sh NAME CMD...
# copies tools/lab/build/libshv_NAME.so over the package library for the
# duration of CMD (restored afterwards), so python labs import that build.
cd "$(dirname "$0")/../.."
lib=paper_1412_8266_b200/libshv.so
cp $lib /tmp/libshv_saved.so
cp tools/lab/build/libshv_$1.so $lib
shift
"$@"
rc=$?
cp /tmp/libshv_saved.so $lib
exit $rc

// Development shim: print a native backtrace on SIGSEGV, then chain to the previous handler.
// gcc -shared -fPIC -g -o tools/debug/libsegv_trace.so tools/debug/segv_trace.c
// Loaded by tests/conftest.py when SVDK_SEGV_TRACE=<path to the .so> is set.
#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <string.h>
#include <unistd.h>
static struct sigaction prev;
static void handler(int sig, siginfo_t* si, void* ctx) {
    void* frames[64];
    const char msg[] = "\n==== SIGSEGV native backtrace ====\n";
    if (write(2, msg, sizeof msg - 1) < 0) _exit(3);
    int n = backtrace(frames, 64);
    backtrace_symbols_fd(frames, n, 2);
    if (prev.sa_flags & SA_SIGINFO) {
        if (prev.sa_sigaction) prev.sa_sigaction(sig, si, ctx);
    } else if (prev.sa_handler != SIG_DFL && prev.sa_handler != SIG_IGN) {
        prev.sa_handler(sig);
    }
    signal(sig, SIG_DFL);
    raise(sig);
}
void segv_trace_install(void) {
    struct sigaction sa;
    memset(&sa, 0, sizeof sa);
    sa.sa_sigaction = handler;
    sa.sa_flags = SA_SIGINFO | SA_NODEFER;
    sigaction(SIGSEGV, &sa, &prev);
    void* warm[4];
    backtrace(warm, 4);  // load libgcc now, not inside the handler
}

/* LD_PRELOAD helper: prints a native backtrace (lib+offset, resolvable with addr2line against the
 * same build) on SIGSEGV/SIGABRT, then re-raises. Debug aid for host-side crashes on the GPU box. */
#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <string.h>
#include <unistd.h>

static void on_sig(int sig) {
    void* bt[64];
    int n = backtrace(bt, 64);
    const char m[] = "\n[segv_trace] native backtrace:\n";
    write(2, m, sizeof(m) - 1);
    backtrace_symbols_fd(bt, n, 2);
    signal(sig, SIG_DFL);
    raise(sig);
}

__attribute__((constructor)) static void init(void) {
    struct sigaction sa;
    memset(&sa, 0, sizeof(sa));
    sa.sa_handler = on_sig;
    sa.sa_flags = SA_RESETHAND;
    sigaction(SIGSEGV, &sa, 0);
    sigaction(SIGABRT, &sa, 0);
}

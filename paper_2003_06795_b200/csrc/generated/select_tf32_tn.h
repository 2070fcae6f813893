#ifndef SELECT_TF32_TN_H
#define SELECT_TF32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tn_config;

static inline select_tf32_tn_config select_tf32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(4435)) {
        if (n < INT64_C(287)) {
            if (k < INT64_C(992)) {
                if (k < INT64_C(544)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(1109)) {
                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                if (k < INT64_C(167)) {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(118)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2218)) {
                            if (k < INT64_C(91)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(111)) {
                                    if (m < INT64_C(555)) {
                                        if (k < INT64_C(272)) {
                                            if (m < INT64_C(278)) {
                                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        if (m < INT64_C(555)) {
                                            if (m < INT64_C(182)) {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(317)) {
                                                    select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(363)) {
                                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(314)) {
                                if (k < INT64_C(28)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(111)) {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(222)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(744)) {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(139)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(555)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(1109)) {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(1536)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(1630)) {
                            if (m < INT64_C(555)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1087)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(182)) {
                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(278)) {
                if (k < INT64_C(10752)) {
                    if (n < INT64_C(1620)) {
                        if (m < INT64_C(12)) {
                            if (m < INT64_C(6)) {
                                if (m < INT64_C(3)) {
                                    if (k < INT64_C(1620)) {
                                        select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(2)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(2897)) {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(2897)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1145)) {
                                if (k < INT64_C(124)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(405)) {
                                        if (m < INT64_C(139)) {
                                            if (m < INT64_C(70)) {
                                                if (k < INT64_C(227)) {
                                                    select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    if (k < INT64_C(1620)) {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(3072)) {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(6)) {
                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(40)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    if (k < INT64_C(725)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(3)) {
                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(6)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(3259)) {
                    if (m < INT64_C(634)) {
                        if (n < INT64_C(992)) {
                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(287)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(405)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(2535)) {
                            if (k < INT64_C(287)) {
                                if (n < INT64_C(744)) {
                                    if (m < INT64_C(1109)) {
                                        if (k < INT64_C(111)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(111)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(182)) {
                                                select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(203)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(1792)) {
                                    if (k < INT64_C(725)) {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(1449)) {
                                            if (n < INT64_C(1449)) {
                                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (n < INT64_C(46)) {
            if (m < INT64_C(70960)) {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(30)) {
                        select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(8870)) {
                            if (k < INT64_C(167)) {
                                if (n < INT64_C(28)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(167)) {
                                if (k < INT64_C(118)) {
                                    if (m < INT64_C(17740)) {
                                        if (k < INT64_C(56)) {
                                            select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(17740)) {
                                        if (n < INT64_C(28)) {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(118)) {
                        select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            }
        } else {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(222)) {
                    if (m < INT64_C(8870)) {
                        if (n < INT64_C(91)) {
                            if (k < INT64_C(385)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(768)) {
                                    select_tf32_tn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(111)) {
                            if (k < INT64_C(32)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(194)) {
                                    select_tf32_tn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (k < INT64_C(3259)) {
                        if (k < INT64_C(1630)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(363)) {
                                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(7168)) {
                            select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(385)) {
                    select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(182)) {
                        if (m < INT64_C(70960)) {
                            if (n < INT64_C(91)) {
                                select_tf32_tn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(91)) {
                                select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(141920)) {
                                    if (k < INT64_C(815)) {
                                        select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_tn_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_TF32_TN_H */
